# build, full GPU suite, latency calibration, quick perf (cfg1 16x29, cfg2 0.3 32x32, cfg0 auto)
OUT=gpurun_out/check.log; : > $OUT
python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -4 >> $OUT
timeout 600 python tools/lat_calibrate.py > gpurun_out/lat_check.jsonl 2>> $OUT
for i in 1 2; do
  timeout 300 python tools/quick_perf.py 1 1.0 16x29 2>&1 | grep gcups >> $OUT
  timeout 300 python tools/quick_perf.py 2 0.3 32x32 2>&1 | grep gcups >> $OUT
  timeout 300 python tools/quick_perf.py 0 1.0 2>&1 | grep gcups >> $OUT
done
if [ -n "$EXTRA" ]; then eval "$EXTRA" >> $OUT 2>&1; fi
cat $OUT
