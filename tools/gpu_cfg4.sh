set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tests/report_configs.py 4 > gpurun_out/c4_configs.jsonl 2> gpurun_out/c4_configs.err; cat gpurun_out/c4_configs.jsonl; tail -2 gpurun_out/c4_configs.err
timeout 900 python tools/quick_perf.py 4 1.0 32x29,32x30,32x32,16x29 > gpurun_out/c4_qp.log 2>&1; cat gpurun_out/c4_qp.log
