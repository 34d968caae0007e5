export PYTHONUNBUFFERED=1
python - <<'PY' > gpurun_out/bg.txt 2>&1
import cProfile, pstats, sys, os, torch
sys.path.insert(0, '.')
import paper_1510_04591_b200 as hb
T, cfg = hb.gen_toeplitz(10000), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
hb.adc_solve(T, cfg); hb.adc_solve(T, cfg); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable(); hb.adc_solve(T, cfg); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(38)
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
PY
cat gpurun_out/bg.txt
