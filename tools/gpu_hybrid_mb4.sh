(cd microbench && timeout 300 ./hybrid_cell > ../gpurun_out/hybrid_mb4.jsonl 2>&1); grep -E "var" gpurun_out/hybrid_mb4.jsonl | grep -E "dpx|hybA_int_imad\"|hybC|hybAC"
