python -c "import __graft_entry__ as g; g.build()" || exit 1
for M in ${MODES:-0 1 2}; do
  echo "QPM=$M"
  SWDB_QPM=$M timeout 900 python -m pytest tests -q -x -m gpu -k "every_tile or config0 or random_small or saturation" 2>&1 | tail -2
  SWDB_QPM=$M timeout 600 python tools/quick_perf.py 1 1.0 ${TILES:-16x29,32x15,32x16,16x32,16x24,32x29} 2>&1
done
