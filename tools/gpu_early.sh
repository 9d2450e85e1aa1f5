# EARLY latency tiles: full GPU suite, latency calibration with and without EARLY
OUT=gpurun_out/early.log; : > $OUT
python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -4 >> $OUT
timeout 600 python tools/lat_calibrate.py > gpurun_out/lat_early1.jsonl 2>> $OUT
SW_DEFS=SW_EARLY=0 python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1
timeout 600 python tools/lat_calibrate.py > gpurun_out/lat_early0.jsonl 2>> $OUT
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
cat $OUT
