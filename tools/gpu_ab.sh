# A/B of build variants: VARIANTS="SW_DEFS=...;SW_DEFS=..." (first = default build);
# parity subset per variant, then pass-kernel GCUPS on TILES1 (cfg1) and TILES2 (cfg2 at 0.3).
# Output: gpurun_out/ab.log
OUT=gpurun_out/ab.log; : > $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "default" "${VS[@]}"; do
  if [ "$v" != "default" ]; then env $v python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || { echo "build failed: $v" >> $OUT; continue; };
  else python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1; fi
  echo "== $v" >> $OUT
  timeout 900 python -m pytest tests -q -x -m gpu -k "${TESTK:-random_small or extreme or every_tile or config0 or streamed}" 2>&1 | tail -1 >> $OUT
  for i in ${REPS:-1}; do
    timeout 300 python tools/quick_perf.py 1 1.0 ${TILES1:-16x29} 2>&1 | grep gcups >> $OUT
    timeout 300 python tools/quick_perf.py 2 0.3 ${TILES2:-32x32} 2>&1 | grep gcups >> $OUT
  done
  if [ -n "$EXTRA" ]; then eval "$EXTRA" >> $OUT 2>&1; fi
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
cat $OUT
