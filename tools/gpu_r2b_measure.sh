# Round 2 (second half) measurement of the current tree (one GPU): GPU suite, smoke, bench
# (default + reference arm + configs[2] strong at one rank), ncu launch list
# and full capture of the pass kernel in the bench configuration, every
# BASELINE configuration with clocks (report_configs), streamed database.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/n_pytest.log; cat gpurun_out/n_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n_smoke.log 2>&1; tail -1 gpurun_out/n_smoke.log
timeout 600 python bench.py > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; cat gpurun_out/n_bench.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/n_bench_ref.json 2>&1; tail -1 gpurun_out/n_bench_ref.json
timeout 900 python bench.py --config 2 --dist --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/n_bench_cfg2.json 2> gpurun_out/n_bench_cfg2.err; cat gpurun_out/n_bench_cfg2.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/n_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launches.csv $CMD > gpurun_out/n_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw16_pass -s 4 -c 1 -o gpurun_out/n_prof_bench $CMD > gpurun_out/n_ncu_full.log 2>&1
tail -2 gpurun_out/n_ncu_full.log
timeout 1800 python tests/report_configs.py 0 1 2 4 --reps 5 > gpurun_out/n_configs.jsonl 2> gpurun_out/n_configs.err; cat gpurun_out/n_configs.jsonl; tail -2 gpurun_out/n_configs.err
timeout 2400 python tests/report_configs.py 3 --reps 5 --batch > gpurun_out/n_cfg3.jsonl 2> gpurun_out/n_cfg3.err; tail -3 gpurun_out/n_cfg3.jsonl; tail -2 gpurun_out/n_cfg3.err
timeout 900 python tools/run_streamed.py 2 128,256,1024 > gpurun_out/n_streamed.jsonl 2>&1; cat gpurun_out/n_streamed.jsonl
timeout 900 python tools/rows_perf.py > gpurun_out/n_rows_mode.jsonl 2>&1; tail -2 gpurun_out/n_rows_mode.jsonl | cut -c1-300
timeout 900 python tools/lat_calibrate.py > gpurun_out/n_lat_calibration.jsonl 2>&1; grep cfg0 gpurun_out/n_lat_calibration.jsonl | head -2
