# Round 2, first GPU pass: whole GPU suite, bench default line, bench configs[2]
# strong scaling at one rank (NCCL gather path), smoke.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/r2a_pytest.log; cat gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; tail -1 gpurun_out/r2a_smoke.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; cat gpurun_out/r2a_bench.json; tail -3 gpurun_out/r2a_bench.err
timeout 900 python bench.py --config 2 --dist --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_cfg2.json 2> gpurun_out/r2a_bench_cfg2.err; cat gpurun_out/r2a_bench_cfg2.json; tail -3 gpurun_out/r2a_bench_cfg2.err
