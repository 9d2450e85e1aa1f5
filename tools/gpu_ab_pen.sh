# A/B: penalty words by shuffle (SW_PENSHFL=1, default) vs IMAD (0); tests; bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 600 python tools/quick_perf.py 1 1.0 16x29,16x30 > gpurun_out/qp_pen1.log 2>&1; cat gpurun_out/qp_pen1.log
timeout 600 python tools/quick_perf.py 2 0.3 32x32,32x31 > gpurun_out/qp2_pen1.log 2>&1; cat gpurun_out/qp2_pen1.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pen1.json 2>&1; tail -1 gpurun_out/bench_pen1.json | cut -c1-400
SW_PENSHFL=0 python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 600 python tools/quick_perf.py 1 1.0 16x29,16x30 > gpurun_out/qp_pen0.log 2>&1; cat gpurun_out/qp_pen0.log
timeout 600 python tools/quick_perf.py 2 0.3 32x32,32x31 > gpurun_out/qp2_pen0.log 2>&1; cat gpurun_out/qp2_pen0.log
