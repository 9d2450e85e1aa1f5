# A/B build variants on cfg1 (16x29) and cfg2 0.3 (32x32), with a parity subset per variant:
# VARIANTS="ENV=.. ENV=..;..."
set -x
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "default" "${VS[@]}"; do
  if [ "$v" != "default" ]; then env $v python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; };
  else python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || exit 1; fi
  echo "== $v"
  timeout 600 python -m pytest tests -q -x -m gpu -k "${TESTK:-random_small or extreme or every_tile or streamed or batch or config0}" 2>&1 | tail -1
  timeout 300 python tools/quick_perf.py 1 1.0 16x29 2>&1 | grep gcups
  timeout 300 python tools/quick_perf.py 2 0.3 32x32 2>&1 | grep gcups
  if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
done
python -m paper_1702_07195_b200.build --force > /dev/null 2>&1
