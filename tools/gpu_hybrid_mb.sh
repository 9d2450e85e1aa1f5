# hybrid fp16/DPX cell microbenchmark + GPU tests on the current tree
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
(cd microbench && timeout 120 ./hybrid_cell > ../gpurun_out/hybrid_mb.jsonl 2>&1); cat gpurun_out/hybrid_mb.jsonl
(cd microbench && timeout 300 ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fp16.sum,sm__inst_executed.sum,sm__pipe_alu_cycles_active.sum,sm__pipe_fma_cycles_active.sum,sm__pipe_fp16_cycles_active.sum,sm__cycles_elapsed.max --clock-control none --csv --log-file ../gpurun_out/hybrid_ncu.csv ./hybrid_cell > /dev/null 2>&1)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
