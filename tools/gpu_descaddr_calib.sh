# calibration of every throughput tile with the descriptor address from s_desc (0) and from s_qp (1)
OUT=gpurun_out/descaddr.log; : > $OUT
for v in 0 1; do
  SW_DEFS=SW_DESCADDR=$v python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || { echo "build $v failed" >> $OUT; continue; }
  timeout 1200 python tools/calibrate_tiles.py 1.0 > gpurun_out/calib_da$v.jsonl 2>> $OUT
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
wc -l gpurun_out/calib_da*.jsonl >> $OUT
cat $OUT
