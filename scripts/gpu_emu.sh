# softmax exponential split: timing of the tile kernel per EVA_SOFTMAX_EMU, and parity with emu
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for e in -1 0 1 2; do echo "== EVA_SOFTMAX_EMU=$e"; EVA_SOFTMAX_EMU=$e python scripts/time_prefill.py tile; done
EVA_SOFTMAX_EMU=1 timeout 600 python -m pytest tests -q -m gpu --timeout 300 -x -k "prefill" 2>&1 | tail -3
EVA_SOFTMAX_EMU=2 timeout 600 python -m pytest tests -q -m gpu --timeout 300 -x -k "prefill_parity or full_size" 2>&1 | tail -3
python scripts/trace_tile.py 1 16 2048 64 64 128 > gpurun_out/trace_cfg2b.txt 2>&1
