# profile the pass kernel for given tiles: TILES env, CFG env
python -c "import __graft_entry__ as g; g.build()" || exit 1
CMD="python tools/quick_perf.py ${CFG:-1} ${SCALE:-0.25} ${TILES:-16x29,32x15}"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && cat gpurun_out/prof_plain.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw16_pass -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof_tiles} $CMD > gpurun_out/ncu_tiles.log 2>&1
tail -2 gpurun_out/ncu_tiles.log
