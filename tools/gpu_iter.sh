# quick iteration: build, GPU parity tests, quick perf on cfg1
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py 1 1.0 ${TILES:-16x29,32x15,32x16,16x32,8x18} > gpurun_out/quick_perf.log 2>&1; cat gpurun_out/quick_perf.log
