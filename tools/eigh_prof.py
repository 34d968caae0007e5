"""Where adc_solve spends its time: python tools/eigh_prof.py cfg N  (cfg in 1, 2, 3, 5)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402

cfg_id, n = sys.argv[1], int(sys.argv[2])
if cfg_id == "1":
    T, cfg = hb.gen_uniform(n, 0), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "2":
    T, cfg = hb.gen_toeplitz(n), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "3":
    T, cfg = hb.gen_kac(n) if hasattr(hb, "gen_kac") else hb.gen_clement(n), hb.SolverConfig(rank_eps=1e-13)
else:
    T, cfg = hb.gen_config5(n, 0), hb.SolverConfig(rank_eps=1e-13)
meth = os.environ.get("HSSEIG_METHOD")
if meth:
    cfg.method = meth
hb.adc_solve(T, cfg)   # warm-up
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = hb.adc_solve(T, cfg)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0, "merges", len(res.merges),
      "hss", sum(m.used_hss for m in res.merges), "peak GB", torch.cuda.max_memory_allocated() / 1e9)
if os.environ.get("HSSEIG_NOPROF") is None:
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
