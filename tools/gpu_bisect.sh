# run one GPU test under several build variants: TEST=..., VARIANTS="A=1;B=0 C=1"
python -c "import __graft_entry__ as g; g.build()" || exit 1
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "default" "${VS[@]}"; do
  if [ "$v" != "default" ]; then env $v python -m paper_1702_07195_b200.build --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }; fi
  echo "== $v"
  timeout 600 python -m pytest tests -q -x -m gpu -k "${TEST}" 2>&1 | grep -E "Error|assert|passed|failed" | head -8
done
