mkdir -p gpurun_out
python scripts/trace_tile.py 1 16 2048 64 64 128 > gpurun_out/trace_cfg1.txt 2>&1
EVA_TRACE_MID=254 python scripts/trace_tile.py 1 16 2048 64 64 128 > gpurun_out/trace_cfg1_last.txt 2>&1
python scripts/time_prefill.py > gpurun_out/time_prefill.txt 2>&1
