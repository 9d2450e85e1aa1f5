# world-2 real-kernel test, GPU suite on the calibrated instantiations, cfg0 launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -k world2 2>&1 | tail -30 > gpurun_out/d_world2.log; tail -5 gpurun_out/d_world2.log
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/d_pytest.log; tail -3 gpurun_out/d_pytest.log
timeout 120 python tools/cfg_launches.py > gpurun_out/d_cfg0.json 2>&1; cat gpurun_out/d_cfg0.json
REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_cfg0_launches.csv python tools/cfg_launches.py > gpurun_out/d_cfg0_ncu.log 2>&1; tail -2 gpurun_out/d_cfg0_ncu.log
