# Official measurement of the current tree: GPU tests, smoke, bench (default
# config, CPU baseline), launch list, ncu --set full of the pass kernel in the
# bench configuration, BASELINE configs 0/1/2/4 with sampled oracle parity.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/fm_pytest.log; cat gpurun_out/fm_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fm_smoke.log 2>&1; tail -1 gpurun_out/fm_smoke.log
timeout 600 python bench.py > gpurun_out/fm_bench.json 2> gpurun_out/fm_bench.err; cat gpurun_out/fm_bench.json; tail -3 gpurun_out/fm_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fm_bench_ref.json 2>&1; tail -1 gpurun_out/fm_bench_ref.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/fm_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fm_launches.csv $CMD > gpurun_out/fm_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw16_pass -s 4 -c 1 -o gpurun_out/fm_prof_bench $CMD > gpurun_out/fm_ncu_full.log 2>&1
tail -2 gpurun_out/fm_ncu_full.log
timeout 1500 python tests/report_configs.py 0 1 2 4 > gpurun_out/fm_configs.jsonl 2> gpurun_out/fm_configs.err; cat gpurun_out/fm_configs.jsonl; tail -3 gpurun_out/fm_configs.err
