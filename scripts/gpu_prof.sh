# build, tests, bench, launch list, ncu full captures of each hot kernel at its config; the
# summaries are written on the box and only the prefill_cfg2 / bwd_main reports come back
# (gpurun returns at most 64 MiB of gpurun_out/)
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -5
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick > /dev/null 2>&1
for k in prefill_cfg3:prefill_sm100_kernel decode_cfg4:decode_kernel summarize_cfg3:summarize prefill_cfg2:prefill_sm100_kernel; do
  w=${k%%:*}; pat=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 -o gpurun_out/prof_${w}_${TAG} -f \
      python scripts/prof_kernels.py $w 2 > gpurun_out/ncu_${w}.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_main_sm100 -s 1 -c 1 -o gpurun_out/prof_bwd_main_${TAG} -f \
    python scripts/prof_backward.py > gpurun_out/ncu_bwd.log 2>&1
for w in prefill_cfg3 decode_cfg4 summarize_cfg3 prefill_cfg2 bwd_main; do
  python scripts/ncu_summary.py gpurun_out/prof_${w}_${TAG}.ncu-rep > gpurun_out/sum_${w}_${TAG}.txt 2>&1
done
python scripts/make_traffic.py ${TAG} > /dev/null 2>&1 && cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_${TAG}.json
rm -f gpurun_out/prof_summarize_cfg3_${TAG}.ncu-rep gpurun_out/prof_decode_cfg4_${TAG}.ncu-rep gpurun_out/prof_prefill_cfg3_${TAG}.ncu-rep
timeout 300 python scripts/time_variants.py > gpurun_out/variants_${TAG}.jsonl 2>&1
ls gpurun_out; du -sh gpurun_out
