for c in 0 16 37 74 148; do echo "== EVA_OVERLAP_SUMM_CTAS=$c"; EVA_OVERLAP_SUMM_CTAS=$c timeout 120 python scripts/time_prefill.py separate 2>&1 | tail -2; done
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "prefill_parity or full_size or sharded or host_pipeline or overlap" 2>&1 | tail -2
