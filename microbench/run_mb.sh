set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
cd microbench
(nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > ../gpurun_out/mb_clocks.csv &) 
./dpx_microbench > ../gpurun_out/mb.jsonl 2>&1 && \
ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed.sum,sm__pipe_alu_cycles_active.sum,sm__pipe_fma_cycles_active.sum,sm__cycles_elapsed.max --clock-control none --csv --log-file ../gpurun_out/mb_ncu.csv ./dpx_microbench > ../gpurun_out/mb_ncu_stdout.log 2>&1
echo done
