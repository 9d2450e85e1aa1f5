# ncu --set full of the first sw32_kernel launch of a cfg4 search
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
CFG=4 REPS=1 B2B=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw32_kernel -s 0 -c 6 -o gpurun_out/s32_prof python tools/cfg_launches.py > gpurun_out/s32_ncu.log 2>&1
tail -3 gpurun_out/s32_ncu.log
ncu -i gpurun_out/s32_prof.ncu-rep --page raw --csv > gpurun_out/s32_raw.csv 2>/dev/null
ncu -i gpurun_out/s32_prof.ncu-rep --page source --csv > gpurun_out/s32_source.csv 2>/dev/null
ls -la gpurun_out/s32_*
