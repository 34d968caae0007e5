"""ADC1 vs ADC2 on BASELINE config 2 (Toeplitz N=10000, leaf 64, tol 1e-13): wall-s and accuracy."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402


def run(n, method, reps=3):
    T = hb.gen_toeplitz(n)
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13, method=method)
    hb.adc_solve(T, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = hb.adc_solve(T, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ref = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    Q = res.Q
    orth = float((Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max()) / n
    hm = [m for m in res.merges if m.used_hss]
    fb = sum(m.fell_back for m in res.merges)
    print(f"{method:10s} N={n} wall {min(ts):.4f} s  hss_merges {len(hm)} fallbacks {fb} "
          f"max_rank {max((m.hss_rank for m in hm), default=0)} eig_err {np.abs(res.lam - ref).max():.2e} "
          f"orth {orth:.2e} top={res.merges[-1]}", flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    for m in ("adc-rand", "adc-srrsc", "dense-dc"):
        run(n, m)
