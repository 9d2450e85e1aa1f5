# streamed database: per-search inputs by copy engine (0) or by a kernel reading the pinned slot (1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -m gpu -k "stream" 2>&1 | tail -4 > gpurun_out/sk_pytest.log; cat gpurun_out/sk_pytest.log
: > gpurun_out/sk_ab.log
for sk in 1 0; do
  echo "== SWDB_STAGE_KERNEL=$sk" >> gpurun_out/sk_ab.log
  SWDB_STAGE_KERNEL=$sk timeout 900 python tools/run_streamed.py 2 128,256,1024 >> gpurun_out/sk_ab.log 2>&1
done
cat gpurun_out/sk_ab.log
