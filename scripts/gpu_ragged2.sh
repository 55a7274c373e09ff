timeout 300 python - <<'PY'
import sys, torch, statistics
sys.path.insert(0, '.')
import bench, paper_2511_00576_b200 as eva
class A: quick = False; steps = 50
r = bench.bench_decode(A(), eva, torch, torch.device('cuda:0'), torch.cuda.current_stream(), 0, 1, bench.load_peaks())
print({k: r[k] for k in ('ms_per_token', 'decode_ms_per_token', 'two_launch_ms_per_token', 'ragged_ms_per_token', 'ragged_hbm_frac')}, r['roofline']['frac'])
PY
timeout 600 python -m pytest tests/test_ragged_gpu.py tests/test_decode_scale_gpu.py -q -m gpu 2>&1 | tail -2
