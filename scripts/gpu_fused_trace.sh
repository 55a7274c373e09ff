mkdir -p gpurun_out
for a in "8 32 8192 128 64 256" "1 16 2048 64 64 128"; do
  echo "== trace $a fused"; timeout 120 python scripts/trace_tile.py $a fused 2>&1 | grep -E 'SUM|flag|EPI|===' | head -60
done > gpurun_out/fused_trace.txt
cat gpurun_out/fused_trace.txt | head -50
