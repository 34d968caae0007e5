"""Full tridiagonal eigendecomposition wall time on the GPU for BASELINE configs 1-3 (and 5 at a given N).

python tools/eigh_bench.py [cfg ...]   cfg in {1, 2, 3, 5, 5:N}
Prints one JSON line per config with wall-s, merge statistics and accuracy metrics
(orthogonality max|Q^T Q - I|/N, residual max|TQ - Q Lambda|/(N max|T|), eigenvalue
error against the closed form where one exists).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402


def metrics(T, lam, Q):
    n = T.n
    nrm = T.norm_max()
    a = torch.as_tensor(T.a, device="cuda")
    b = torch.as_tensor(T.b, device="cuda")
    lamd = torch.as_tensor(lam, device="cuda")
    TQ = a[:, None] * Q
    TQ[:-1] += b[:, None] * Q[1:]
    TQ[1:] += b[:, None] * Q[:-1]
    res = float((TQ - Q * lamd[None, :]).abs().max()) / (n * nrm)
    del TQ
    G = Q.T @ Q
    G.diagonal().sub_(1.0)
    orth = float(G.abs().max()) / n
    del G
    return orth, res


def run(name, T, cfg, exact=None, reps=2):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = hb.adc_solve(T, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    orth, resid = metrics(T, res.lam, res.Q)
    line = {"config": name, "N": T.n, "wall_s": best, "method": cfg.method,
            "leaf_size": cfg.leaf_size, "hss_threshold": cfg.hss_threshold,
            "rank_eps": cfg.rank_eps, "merges": len(res.merges),
            "hss_merges": sum(m.used_hss for m in res.merges),
            "fallbacks": sum(m.fell_back for m in res.merges),
            "top_kept": res.merges[-1].kept if res.merges else 0,
            "orthogonality": orth, "residual": resid, "flops": res.flops.as_dict()}
    if exact is not None:
        line["eig_err_over_normT"] = float(np.abs(res.lam - exact).max()) / T.norm_max()
    print(json.dumps(line), flush=True)
    del res
    torch.cuda.empty_cache()


def main():
    which = sys.argv[1:] or ["1", "2", "3"]
    for w in which:
        if w == "1":
            T = hb.gen_uniform(2000, 0)
            run("cfg1_uniform_N2000", T, hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13))
        elif w == "2":
            n = 10000
            T = hb.gen_toeplitz(n)
            exact = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
            run("cfg2_toeplitz_N10000_adc2", T, hb.SolverConfig(leaf_size=64, hss_threshold=256,
                                                                rank_eps=1e-13), exact)
        elif w == "3":
            n = 20000
            T = hb.gen_kac(n)
            run("cfg3_kac_N20000", T, hb.SolverConfig(rank_eps=1e-13), -(n - 1) + 2.0 * np.arange(n))
        elif w.startswith("5"):
            n = int(w.split(":")[1]) if ":" in w else 65536
            T = hb.gen_config5(n, 0)
            run(f"cfg5_N{n}", T, hb.SolverConfig(rank_eps=1e-13), reps=1)


if __name__ == "__main__":
    main()
