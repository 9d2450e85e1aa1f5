(cd microbench && timeout 200 ./hybrid_cell > ../gpurun_out/hybrid_mb3.jsonl 2>&1); grep -E "var" gpurun_out/hybrid_mb3.jsonl | grep -E "dpx|hybA"
