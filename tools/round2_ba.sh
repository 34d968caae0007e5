export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "srrsc or adc1 or baseline" 2>&1 | tail -2
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_1510_04591_b200 as hb
T = hb.gen_toeplitz(10000)
for meth in ("adc-srrsc", "adc-rand"):
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13, method=meth)
    hb.adc_solve(T, cfg); hb.adc_solve(T, cfg)
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter(); hb.adc_solve(T, cfg); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(meth, f"{best*1e3:.2f} ms")
PY
