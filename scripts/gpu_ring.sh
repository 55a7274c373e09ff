python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
python - <<'PY'
import torch, ctypes
import paper_2511_00576_b200 as eva
PY
for r in 0 32 54; do echo "== EVA_PREFILL_RING=$r"; EVA_PREFILL_RING=$r python scripts/time_prefill.py tile; done
EVA_PREFILL_RING=32 timeout 600 python -m pytest tests -q -m gpu --timeout 300 -x -k "prefill" 2>&1 | tail -2
EVA_PREFILL_RING=54 timeout 600 python -m pytest tests -q -m gpu --timeout 300 -x -k "prefill" 2>&1 | tail -2
