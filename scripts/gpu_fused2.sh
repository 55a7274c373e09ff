mkdir -p gpurun_out
for o in 0 1; do echo "== EVA_FUSED_ORDER=$o"; EVA_FUSED_ORDER=$o timeout 300 python scripts/time_prefill.py fused 2>&1 | tail -2; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_sm100 -s 3 -c 1 -o gpurun_out/prof_fused -f \
    python scripts/time_prefill.py fused > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/sum_fused.txt 2>&1
head -9 gpurun_out/sum_fused.txt
timeout 120 python scripts/trace_tile.py 8 32 8192 128 64 256 fused 2>&1 | grep -E 'SUM|flag|EPI|===' | head -40
