for A in 0 1 2; do
  SW_ABLATE=$A python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || echo "build $A failed"
  echo "ABLATE=$A"
  timeout 300 python tools/quick_perf.py 1 1.0 16x29,32x15,32x16 2>&1 | grep gcups
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
