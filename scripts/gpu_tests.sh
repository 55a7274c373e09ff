mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -8 > gpurun_out/tests_full.txt
cat gpurun_out/tests_full.txt
timeout 300 python scripts/time_prefill.py 2>&1 | tail -8
