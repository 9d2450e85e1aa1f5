# per-pipe instruction counts of the bench's pass kernel (for roofline I_pipe)
python -c "import __graft_entry__ as g; g.build()" || exit 1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/ip_plain.log 2>&1 && \
timeout 900 ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_lsu.sum,smsp__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg,gpu__time_duration.sum --clock-control none -k regex:sw16_pass -s 4 -c 1 --csv $CMD > gpurun_out/ip_ncu.csv 2> gpurun_out/ip_ncu.err
grep -E "sw16_pass" gpurun_out/ip_ncu.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
