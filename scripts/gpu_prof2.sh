mkdir -p gpurun_out
for k in prefill_cfg3:prefill_sm100_kernel summarize_cfg3:summarize prefill_cfg2:prefill_sm100_kernel; do
  w=${k%%:*}; pat=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 -o gpurun_out/prof_${w}_r02 -f \
      python scripts/prof_kernels.py $w 2 > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_${w}_r02.ncu-rep > gpurun_out/sum_${w}_r02.txt 2>&1
  python scripts/sass_stalls.py gpurun_out/prof_${w}_r02.ncu-rep 30 > gpurun_out/stalls_${w}_r02.txt 2>&1
done
ls -la gpurun_out/*r02*
