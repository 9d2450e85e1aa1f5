set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --config 3 --scale 0.02 --steps 2 --warmup 3 --no-cpu-baseline 2> gpurun_out/c3.err | cut -c1-600; tail -2 gpurun_out/c3.err
timeout 600 python bench.py --config 4 --scale 0.1 --steps 2 --warmup 3 --no-cpu-baseline 2> gpurun_out/c4.err | cut -c1-400; tail -2 gpurun_out/c4.err
timeout 600 python bench.py --config 0 --dist --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/c0.err | cut -c1-400; tail -2 gpurun_out/c0.err
