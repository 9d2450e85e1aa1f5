# A/B of the pass-kernel arithmetic: SW_ARITH=1 (biased, default) vs 0 (relu DPX)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
TL=${TILES:-16x29,32x29,16x32,32x32,16x24,8x18}
timeout 600 python tools/quick_perf.py 1 1.0 $TL > gpurun_out/qp_arith1.log 2>&1; cat gpurun_out/qp_arith1.log
timeout 600 python tools/quick_perf.py 4 0.25 32x29 > gpurun_out/qp4_arith1.log 2>&1; cat gpurun_out/qp4_arith1.log
SW_ARITH=0 python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 600 python tools/quick_perf.py 1 1.0 $TL > gpurun_out/qp_arith0.log 2>&1; cat gpurun_out/qp_arith0.log
