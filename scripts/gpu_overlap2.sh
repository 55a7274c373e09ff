for c in 0 1 2 3; do echo "EVA_SUMM_PER_SM=$c"; EVA_SUMM_PER_SM=$c python scripts/time_overlap.py 2>&1 | grep "T=2048"; done
