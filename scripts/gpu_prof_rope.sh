TAG=${TAG:-r02o}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_sm100 -s 1 -c 1 -o gpurun_out/prof_prefill_ropeq_configs2_${TAG} -f \
    python scripts/prof_kernels.py prefill_ropeq_configs2 2 > gpurun_out/ncu_ropeq.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:summarize_bulk -s 1 -c 1 -o gpurun_out/prof_summarize_rope_configs2_${TAG} -f \
    python scripts/prof_kernels.py summarize_rope_configs2 2 > gpurun_out/ncu_srope.log 2>&1
for w in prefill_ropeq_configs2 summarize_rope_configs2; do
  python scripts/ncu_summary.py gpurun_out/prof_${w}_${TAG}.ncu-rep > gpurun_out/sum_${w}_${TAG}.txt 2>&1
  python scripts/sass_stalls.py gpurun_out/prof_${w}_${TAG}.ncu-rep 20 > gpurun_out/stalls_${w}_${TAG}.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/sum_*_${TAG}.txt
