mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 python scripts/trace_dual.py 8 32 8192 128 64 256 640 > gpurun_out/trace_dual.txt 2>&1
tail -3 gpurun_out/trace_dual.txt
