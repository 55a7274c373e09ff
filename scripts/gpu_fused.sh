# fused-summary prefill: timing, traces, ncu of the fused kernel, then parity (bounded by timeouts)
mkdir -p gpurun_out
timeout 300 python scripts/time_prefill.py 2>&1 | tail -8
for a in "8 32 8192 128 64 256" "1 16 2048 64 64 128"; do
  echo "== trace $a fused"; timeout 120 python scripts/trace_tile.py $a fused 2>&1 | head -150
done > gpurun_out/fused_trace.txt
grep -E 'SUM|flag|EPI|===' gpurun_out/fused_trace.txt | head -40
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_sm100 -s 3 -c 1 -o gpurun_out/prof_fused -f \
    python scripts/time_prefill.py fused > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/sum_fused.txt 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout 240 -x -k "prefill or fused or sharded or full_size or long_context" 2>&1 | tail -15 > gpurun_out/fused_tests.txt
tail -3 gpurun_out/fused_tests.txt
