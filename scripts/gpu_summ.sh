mkdir -p gpurun_out
timeout 300 python scripts/time_prefill.py summarize_only separate attention_only 2>&1 | tail -6
EVA_SUMMARIZE_REG=1 timeout 300 python scripts/time_prefill.py summarize_only separate 2>&1 | tail -4
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -x -k "summar or cache or decode or rope or proj or ragged or backward" 2>&1 | tail -4
