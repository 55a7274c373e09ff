# One GPU call: build, bench (our arm), launch list, one full ncu capture of the prefill kernel.
set -x
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -c 3000 gpurun_out/bench_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --quick > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefill -s 4 -c 2 -o gpurun_out/prof_prefill_${TAG} -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
ls -la gpurun_out
