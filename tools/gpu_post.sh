mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_bench.py -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; cut -c1-200 gpurun_out/f_bench.json
timeout 900 python tools/wave_small.py > gpurun_out/wave_small.jsonl 2> gpurun_out/wave_small.err; cat gpurun_out/wave_small.jsonl
