# full-size calibration of every throughput tile under build variants:
# VARIANTS="name:DEFS;name:DEFS" (DEFS space-separated, e.g. "SW_DESCADDR=0 SW_ROWAHEAD=0")
OUT=gpurun_out/variant_calib.log; : > $OUT
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  SW_DEFS="$defs" python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || { echo "build $name failed" >> $OUT; continue; }
  timeout 1200 python tools/calibrate_tiles.py 1.0 > gpurun_out/calib_$name.jsonl 2>> $OUT
  echo "$name: $(wc -l < gpurun_out/calib_$name.jsonl) tiles" >> $OUT
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
cat $OUT
