# cell-formulation microbenchmark (microbench/hybrid_cell.cu): cells/clk/SM per variant,
# plus per-pipe instruction counts under ncu
set -x
(cd microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o hybrid_cell hybrid_cell.cu && \
 timeout 300 ./hybrid_cell > ../gpurun_out/hybrid_mb.jsonl 2>&1); cat gpurun_out/hybrid_mb.jsonl
(cd microbench && timeout 600 ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed.sum,sm__pipe_alu_cycles_active.sum,sm__pipe_fma_cycles_active.sum,sm__cycles_elapsed.max --clock-control none --csv --log-file ../gpurun_out/hybrid_ncu.csv ./hybrid_cell > /dev/null 2>&1)
