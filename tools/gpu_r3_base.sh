# re-entry check: build, full GPU suite, smoke, bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/base_pytest.log; cat gpurun_out/base_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err; cut -c1-900 gpurun_out/base_bench.json; tail -2 gpurun_out/base_bench.err
