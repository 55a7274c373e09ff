# ncu full captures of the two tensor-core prefill variants at configs[2] (per-GPU shape)
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for v in pair tile; do
  EVA_PROF_KERNEL=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill -s 1 -c 1 \
     -o gpurun_out/prof_prefill_${v}_${TAG} -f python scripts/prof_kernels.py prefill_cfg3 2 > gpurun_out/ncu_prefill_${v}.log 2>&1
  tail -2 gpurun_out/ncu_prefill_${v}.log
done
