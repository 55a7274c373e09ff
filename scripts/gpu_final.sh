TAG=${TAG:-r02i}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -3 > gpurun_out/tests_${TAG}.txt
cat gpurun_out/tests_${TAG}.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -3 gpurun_out/smoke_${TAG}.txt
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_${TAG}.json 2> gpurun_out/bench_reference_${TAG}.err
tail -c 600 gpurun_out/bench_${TAG}.json
