for v in 0 1; do echo "== EVA_RAGGED_TWO_LAUNCH=$v"; EVA_RAGGED_TWO_LAUNCH=$v timeout 300 python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import bench, paper_2511_00576_b200 as eva
class A: quick = False; steps = 50
for _ in range(2):
    r = bench.bench_decode(A(), eva, torch, torch.device('cuda:0'), torch.cuda.current_stream(), 0, 1, bench.load_peaks())
    print({k: round(r[k], 4) for k in ('ms_per_token', 'ragged_ms_per_token', 'ragged_hbm_frac')})
PY
done
