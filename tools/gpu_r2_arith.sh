# Round 2: biased-unsigned arithmetic with carry propagation (default
# SW_ARITH=2) against the signed one (SW_ARITH=1); compact streamed chunks.
set -x
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -8
timeout 900 python tests/report_configs.py 4 --reps 5 > gpurun_out/r2d_cfg4_arith2.jsonl 2> gpurun_out/r2d_cfg4_arith2.err; cat gpurun_out/r2d_cfg4_arith2.jsonl; tail -2 gpurun_out/r2d_cfg4_arith2.err
timeout 900 python tools/run_streamed.py 2 256,1024 > gpurun_out/r2d_streamed.jsonl 2>&1; cat gpurun_out/r2d_streamed.jsonl
