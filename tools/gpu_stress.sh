# GPU suite, latency calibration, then a randomised stress run against the oracle
OUT=gpurun_out/stress.log; : > $OUT
python -m paper_1702_07195_b200.build --force > /dev/null 2>> $OUT || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2 >> $OUT
timeout 600 python tools/lat_calibrate.py > gpurun_out/lat_calib_final.jsonl 2>> $OUT
timeout ${STRESS_S:-1500} python tests/report_stress.py --seconds ${STRESS_RUN:-1200} --seed ${SEED:-5} > gpurun_out/stress_run.log 2>&1; echo "stress exit $?" >> $OUT
tail -3 gpurun_out/stress_run.log >> $OUT
cat $OUT
