"""Sweep of solver.DENSE_PANEL_MIN_K (merges with at least this many kept poles take the
materialised-panel halves update, the rest the grouped dense tiles) on configs 5 and 1."""
import os, sys, time
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb
from paper_1510_04591_b200 import solver

cases = [("cfg5", hb.gen_config5(65536, 0), hb.SolverConfig(rank_eps=1e-13)),
         ("cfg1", hb.gen_uniform(2000, 0), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)),
         ("cfg5_16k", hb.gen_config5(16384, 0), hb.SolverConfig(rank_eps=1e-13))]
for mk in (192, 256, 384, 512, 768, 1024):
    solver.DENSE_PANEL_MIN_K = mk
    out = []
    for name, T, cfg in cases:
        hb.adc_solve(T, cfg); hb.adc_solve(T, cfg)
        best = 1e9
        for _ in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter(); hb.adc_solve(T, cfg); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        out.append(f"{name} {best * 1e3:.2f} ms")
    print(mk, "  ".join(out))
