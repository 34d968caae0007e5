"""Timing probe: config-2 / config-3 solves with the per-tree flop accounting stubbed out
(how much of the wall is the Python flop loops)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb
from paper_1510_04591_b200 import hss

def run(T, cfg, tag):
    hb.adc_solve(T, cfg); hb.adc_solve(T, cfg)
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter(); hb.adc_solve(T, cfg); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(tag, f"{best*1e3:.2f} ms")

T2, c2 = hb.gen_toeplitz(10000), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
T3, c3 = hb.gen_kac(20000), hb.SolverConfig(rank_eps=1e-13)
run(T2, c2, "cfg2 adc2"); run(T3, c3, "cfg3")
hss._construct_flops = lambda *a, **k: 0
hss.mult_flops = lambda *a, **k: 0
run(T2, c2, "cfg2 adc2 (no flop loops)"); run(T3, c3, "cfg3 (no flop loops)")
