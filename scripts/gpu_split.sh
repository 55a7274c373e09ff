# EVA_PREFILL_SPLIT (8 softmax warps, d = 64): parity, then the configs[1] step with and without
mkdir -p gpurun_out
EVA_PREFILL_SPLIT=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_variants_gpu.py -q -m gpu -x --timeout 300 2>&1 | tail -3
for e in 0 1 0 1; do
  echo "SPLIT=$e $(EVA_PREFILL_SPLIT=$e python bench.py --steps 200 --warmup 10 --no-extras --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"]*1e3, d["breakdown_ms"]["prefill"]*1e3, d["roofline"]["frac"])')"
done
