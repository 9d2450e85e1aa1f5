# A/B build variants on cfg1 (16x29) and cfg2 0.3 (32x32): VARIANTS="ENV=.. ENV=..;..."
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "default" "${VS[@]}"; do
  if [ "$v" != "default" ]; then env $v python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }; fi
  echo "== $v"
  timeout 300 python tools/quick_perf.py 1 1.0 16x29 2>&1 | grep gcups
  timeout 300 python tools/quick_perf.py 2 0.3 32x32 2>&1 | grep gcups
done
