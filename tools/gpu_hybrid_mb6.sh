(cd microbench && timeout 300 ./hybrid_cell > ../gpurun_out/hybrid_mb6.jsonl 2>&1); grep -E "var" gpurun_out/hybrid_mb6.jsonl | grep -E "hybA_int_imad\"|profile16"
