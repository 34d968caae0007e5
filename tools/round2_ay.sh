export PYTHONUNBUFFERED=1
python tools/eigh_prof.py 2 10000 2>&1 | head -40
python - <<'PY'
import cProfile, pstats, sys, os, torch
sys.path.insert(0, '.')
import paper_1510_04591_b200 as hb
T, cfg = hb.gen_toeplitz(10000), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
hb.adc_solve(T, cfg); hb.adc_solve(T, cfg)
pr = cProfile.Profile(); pr.enable(); hb.adc_solve(T, cfg); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
PY
