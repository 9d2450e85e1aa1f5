# Round 2 final measurement of the tree (one GPU): GPU suite, smoke, bench
# (default + reference arm + configs[2] strong at one rank), ncu launch list
# and full capture of the pass kernel in the bench configuration, every
# BASELINE configuration with clocks (report_configs), cfg3 sweep, streamed
# database, launch lists of a cfg0 and a cfg4 search.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/f_pytest.log; cat gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; cat gpurun_out/f_bench.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.json 2>&1; tail -1 gpurun_out/f_bench_ref.json
timeout 900 python bench.py --config 2 --dist --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_cfg2.json 2> gpurun_out/f_bench_cfg2.err; cat gpurun_out/f_bench_cfg2.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/f_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv $CMD > gpurun_out/f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw16_pass -s 4 -c 1 -o gpurun_out/f_prof_bench $CMD > gpurun_out/f_ncu_full.log 2>&1
tail -2 gpurun_out/f_ncu_full.log
timeout 1800 python tests/report_configs.py 0 1 2 4 --reps 5 > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; cat gpurun_out/f_configs.jsonl; tail -2 gpurun_out/f_configs.err
timeout 2400 python tests/report_configs.py 3 --reps 5 --batch > gpurun_out/f_cfg3.jsonl 2> gpurun_out/f_cfg3.err; tail -3 gpurun_out/f_cfg3.jsonl; tail -2 gpurun_out/f_cfg3.err
timeout 900 python tools/run_streamed.py 2 128,256,1024 > gpurun_out/f_streamed.jsonl 2>&1; cat gpurun_out/f_streamed.jsonl
CFG=0 REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_cfg0_launches.csv python tools/cfg_launches.py > gpurun_out/f_cfg0_ncu.log 2>&1
CFG=4 REPS=1 B2B=1 timeout 600 python tools/cfg_launches.py > gpurun_out/f_cfg4.json 2>&1; cat gpurun_out/f_cfg4.json | cut -c1-300
CFG=4 REPS=1 B2B=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_cfg4_launches.csv python tools/cfg_launches.py > gpurun_out/f_cfg4_ncu.log 2>&1
