# GPU suite + a stress run on the current tree
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -6
timeout 900 python tests/report_stress.py --seconds ${STRESS_S:-600} --seed ${SEED:-3} > gpurun_out/v_stress.log 2>&1; tail -3 gpurun_out/v_stress.log
