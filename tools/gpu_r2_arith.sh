# Round 2: the biased-unsigned arithmetic (default SW_ARITH=2) against the
# signed one (SW_ARITH=1): whole GPU suite on the default, bench line, cfg4
# (flagged + s32) and cfg1 under both.
set -x
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests -q -x -m gpu 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench.json
timeout 900 python tests/report_configs.py 4 1 --reps 5 > gpurun_out/r2c_cfg41_arith2.jsonl 2> gpurun_out/r2c_cfg41_arith2.err; cat gpurun_out/r2c_cfg41_arith2.jsonl; tail -2 gpurun_out/r2c_cfg41_arith2.err
SW_ARITH=1 python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 900 python tests/report_configs.py 4 1 --reps 5 > gpurun_out/r2c_cfg41_arith1.jsonl 2> gpurun_out/r2c_cfg41_arith1.err; cat gpurun_out/r2c_cfg41_arith1.jsonl; tail -2 gpurun_out/r2c_cfg41_arith1.err
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
