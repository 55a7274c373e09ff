python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for k in tile pair; do
  echo "== $k"; timeout 120 python scripts/probe_prefill.py $k 2>&1 | tail -12; echo "probe rc=$?"
done
