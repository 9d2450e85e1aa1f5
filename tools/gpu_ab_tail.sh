# A/B of the profile tail layout (kernels.cuh SW_QPTAIL / SW_TAILADDR): parity
# subset + pass-kernel GCUPS on tiles with R % 4 = 1, 2 (and 0 as control).
set -x
for v in "SW_QPTAIL=0" "SW_QPTAIL=1 SW_TAILADDR=0" "SW_QPTAIL=1 SW_TAILADDR=1"; do
  env $v python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  timeout 600 python -m pytest tests -q -x -m gpu -k "random_small or extreme or every_tile or batch_random or wavefront" 2>&1 | tail -1
  for i in 1 2; do
    timeout 300 python tools/quick_perf.py 1 1.0 16x29,32x29,8x29,16x30,16x22,32x32 2>&1 | grep gcups
  done
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
