# tile calibration for NTMODE 0/1 (biased arithmetic) + ncu of the cfg1 16x29 pass kernel
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/calibrate_tiles.py 0.3 > gpurun_out/calib_nt0.jsonl 2>&1
CMD="python tools/quick_perf.py 1 0.5 16x29"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw16_pass -s 3 -c 1 -o gpurun_out/prof_b16x29 $CMD > gpurun_out/ncu_b.log 2>&1
SW_NTMODE=1 python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1
timeout 900 python tools/calibrate_tiles.py 0.3 > gpurun_out/calib_nt1.jsonl 2>&1
paste gpurun_out/calib_nt0.jsonl gpurun_out/calib_nt1.jsonl
