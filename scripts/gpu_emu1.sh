mkdir -p gpurun_out; : > gpurun_out/emu1.txt
for e in 0 1 2 4 -1 0; do
  echo "EMU=$e $(EVA_SOFTMAX_EMU=$e python bench.py --steps 200 --warmup 10 --no-extras --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"]*1e3, d["breakdown_ms"]["prefill"]*1e3, d["roofline"]["frac"])')" >> gpurun_out/emu1.txt
done
cat gpurun_out/emu1.txt
