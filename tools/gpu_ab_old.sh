# same-box A/B of the current tree against an older tree exported to oldlib/ (git archive <rev>)
OUT=gpurun_out/ab_old.log; : > $OUT
python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1
(cd oldlib && python -m paper_1702_07195_b200.build --force > /dev/null 2>&1) || echo "old build failed" >> $OUT
for i in 1 2; do
  echo "== new $i" >> $OUT
  timeout 300 python tools/quick_perf.py 1 1.0 16x29 2>&1 | grep gcups >> $OUT
  timeout 300 python tools/quick_perf.py 2 0.3 32x32,16x29 2>&1 | grep gcups >> $OUT
  echo "== old $i" >> $OUT
  (cd oldlib && timeout 300 python tools/quick_perf.py 1 1.0 16x29 2>&1 | grep gcups) >> $OUT
  (cd oldlib && timeout 300 python tools/quick_perf.py 2 0.3 32x32,16x29 2>&1 | grep gcups) >> $OUT
done
if [ -n "$EXTRA" ]; then eval "$EXTRA" >> $OUT 2>&1; fi
cat $OUT
