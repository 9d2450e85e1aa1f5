set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
(nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_r1a.csv &)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py 1 1.0 16x32,32x16,16x29,32x15,8x20,16x24,32x24 > gpurun_out/quick_perf.log 2>&1
cat gpurun_out/quick_perf.log
