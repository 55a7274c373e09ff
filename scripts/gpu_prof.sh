# build, tests, bench, launch list, ncu full captures of each hot kernel at its BASELINE config
# (0-indexed names); summaries written on the box, large reports dropped before the copy-back
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -3 > gpurun_out/tests_${TAG}.txt
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick --no-extras > /dev/null 2>&1
for k in prefill_configs2:prefill_sm100_kernel decode_configs3:decode_kernel summarize_configs2:summarize prefill_configs1:prefill_sm100_kernel prefill_rope_configs2:prefill_sm100_kernel decode_ragged_configs3:decode_kernel; do
  w=${k%%:*}; pat=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 -o gpurun_out/prof_${w}_${TAG} -f \
      python scripts/prof_kernels.py $w 2 > gpurun_out/ncu_${w}.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_main_sm100 -s 1 -c 1 -o gpurun_out/prof_bwd_main_${TAG} -f \
    python scripts/prof_backward.py > gpurun_out/ncu_bwd.log 2>&1
for w in prefill_configs2 decode_configs3 summarize_configs2 prefill_configs1 prefill_rope_configs2 decode_ragged_configs3 bwd_main; do
  python scripts/ncu_summary.py gpurun_out/prof_${w}_${TAG}.ncu-rep > gpurun_out/sum_${w}_${TAG}.txt 2>&1
  python scripts/sass_stalls.py gpurun_out/prof_${w}_${TAG}.ncu-rep 20 > gpurun_out/stalls_${w}_${TAG}.txt 2>&1
done
python scripts/make_traffic.py ${TAG} > /dev/null 2>&1 && cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_${TAG}.json
rm -f gpurun_out/*.ncu-rep
ls gpurun_out; du -sh gpurun_out
