# the 128-key two-query-tile prefill (prefill_dual.cu): parity tests, then timing against the
# 64-key kernel (EVA_PREFILL_DUAL=0) and over the softmax variants (EVA_DUAL_EMU)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout 120 -x -k "prefill or full_size or sweep or sharded" 2>&1 | tail -3 > gpurun_out/dual_tests.txt
for e in 0 2 -1; do
  echo "EVA_DUAL_EMU=$e" >> gpurun_out/dual_time.txt
  EVA_DUAL_EMU=$e timeout 300 python scripts/time_prefill.py attention_only >> gpurun_out/dual_time.txt 2>&1
done
timeout 120 python scripts/trace_dual.py 8 32 8192 128 64 256 640 > gpurun_out/trace_dual.txt 2>&1
cat gpurun_out/dual_tests.txt gpurun_out/dual_time.txt
