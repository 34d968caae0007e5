"""Orthogonality / residual of the GPU solver vs the oracle (reference restatement) on one matrix."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from oracle import hss_oracle as orc  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "kac"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 64
thr = 4 * leaf
T = {"kac": hb.gen_kac, "toeplitz": hb.gen_toeplitz, "cfg5": lambda m: hb.gen_config5(m, 0),
     "uniform": lambda m: hb.gen_uniform(m, 0)}[fam](n)
for method in ("adc-rand", "dense-dc"):
    cfg = hb.SolverConfig(leaf_size=leaf, hss_threshold=thr, rank_eps=1e-13, method=method)
    t = time.time()
    lam_o, Q_o, info_o, _ = orc.adc_solve(T.a, T.b, orc.Config(leaf_size=leaf, hss_threshold=thr,
                                                                rank_eps=1e-13, method=method))
    to = time.time() - t
    res = hb.adc_solve(T, cfg)
    Qg = res.Q.cpu().numpy()
    print(method, fam, n, "oracle %.1fs" % to,
          "orth oracle %.3e gpu %.3e" % (orc.orthogonality(Q_o), orc.orthogonality(Qg)),
          "resid oracle %.3e gpu %.3e" % (orc.residual(T.a, T.b, lam_o, Q_o), orc.residual(T.a, T.b, res.lam, Qg)),
          "eig diff %.2e" % (np.abs(res.lam - lam_o).max() / T.norm_max()),
          "hss merges", sum(i.used_hss for i in info_o), sum(m.used_hss for m in res.merges), flush=True)
