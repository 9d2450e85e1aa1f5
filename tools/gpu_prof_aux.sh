# ncu --set full of the 32-bit re-scoring kernel (cfg4) and of the wavefront kernel
# (200 long sequences, m = 5478), after plain runs of the same commands
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
C4="python tests/report_configs.py 4 --sample 200 --reps 1"
timeout 600 $C4 > gpurun_out/aux_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:sw32_kernel -s 1 -c 1 -o gpurun_out/prof_sw32 $C4 > gpurun_out/aux_ncu_sw32.log 2>&1
cat > /tmp/wave_one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, sw_inputs as si, paper_1702_07195_b200 as sw
rng = np.random.default_rng(5)
db = si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(20000, 35000, 200)])
sw.sw_db_load(db.residues, db.offsets)
q = si.rr_residues(rng, 5478)
for _ in range(2):
    sw.sw_search(q, si.BLOSUM62, 10, 2)
print(sw.sw_last_stats(), sw.sw_last_timing())
PY
timeout 300 python /tmp/wave_one.py > gpurun_out/aux_wave.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:sw16_pass -s 1 -c 1 -o gpurun_out/prof_wave python /tmp/wave_one.py > gpurun_out/aux_ncu_wave.log 2>&1
tail -1 gpurun_out/aux_c4.log | cut -c1-200; cat gpurun_out/aux_wave.log; tail -1 gpurun_out/aux_ncu_sw32.log; tail -1 gpurun_out/aux_ncu_wave.log
