# streamed database: resident head on / off (SWDB_STREAM_HEAD), streamed tests first
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -m gpu -k "stream" 2>&1 | tail -8 > gpurun_out/hd_pytest.log; cat gpurun_out/hd_pytest.log
: > gpurun_out/hd_ab.log
for hd in 1 0; do
  echo "== SWDB_STREAM_HEAD=$hd" >> gpurun_out/hd_ab.log
  SWDB_STREAM_HEAD=$hd timeout 900 python tools/run_streamed.py 2 64,128,256,512,1024 >> gpurun_out/hd_ab.log 2>&1
done
cat gpurun_out/hd_ab.log
