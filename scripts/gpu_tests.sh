set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -8
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -30
