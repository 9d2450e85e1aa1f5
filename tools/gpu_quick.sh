# build + GPU tests + cfg4 run_configs + cfg1 quick perf
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 900 python tests/report_configs.py ${CFGS:-4} 2>/dev/null | cut -c1-400
