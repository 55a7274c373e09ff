python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 python scripts/trace_prefill.py 8192 8 32 128 > gpurun_out/trace_cfg3.txt 2>&1; tail -25 gpurun_out/trace_cfg3.txt
timeout 300 python -m pytest tests -q -m gpu --timeout 300 -x 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_trace.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/bench_trace.json')); print(j['prefill_configs2']['prefill_ms'], j['prefill_configs2']['roofline']['frac'], j['breakdown_ms'], j['decode_configs3']['decode_ms_per_token'])"
