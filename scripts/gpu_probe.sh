python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 python scripts/probe_prefill.py 2>&1 | tail -20
echo "probe rc=$?"
