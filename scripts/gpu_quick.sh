# build, the given pytest selection, tile traces, bench (no extras)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -5
python scripts/trace_tile.py 1 16 2048 64 64 128 > gpurun_out/trace_cfg2.txt 2>&1
python scripts/trace_tile.py 8 32 8192 128 64 256 > gpurun_out/trace_cfg3.txt 2>&1
python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -c 1500 gpurun_out/bench_quick.json
