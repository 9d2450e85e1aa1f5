# Round 2 (last session) check of the tree: GPU suite, smoke, bench, then the
# row-order variant calibration (tools/gpu_variant_calib.sh) at full size.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/c_pytest.log; cat gpurun_out/c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; tail -1 gpurun_out/c_smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; cat gpurun_out/c_bench.json
VARIANTS="ahead:SW_ROWAHEAD=1;plain:SW_ROWAHEAD=0" bash tools/gpu_variant_calib.sh
