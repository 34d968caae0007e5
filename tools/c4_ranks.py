"""Per-level ranks of the config-4 tree (offdiag and reference samples) and per-level
multiply time (CUDA events): python tools/c4_ranks.py [N]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200 import hss  # noqa: E402
from paper_1510_04591_b200.matgen import isolated_merge_system  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d, u, rho = isolated_merge_system(N, 0)
sys_ = hb.RankOneSystem(d, u, rho)
sol = hb.solve_secular(sys_)
hb.recompute_weights(d, sol, u, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(sys_, sol)
part = hb.build_partition(N, 128, C.d, C.gamma, C.mu)
r = min(hb.estimate_rank(part, C.d, C.gamma, C.mu, 1e-13, 100), part.min_leaf - 10)
print("N", N, "r", r, "w", r + 10, "leaves", part.n_leaves)
X = torch.randn(N, N, dtype=torch.float64, device="cuda")
for offdiag in (True, False):
    H = hb.rand_hss_construct(C, part, r, p=10, seed=[0, 0], offdiag=offdiag)
    rU, rV = H.ranks()
    print(f"offdiag={offdiag} rmax={H.ct.rmax} ws={H.ct.ws}")
    for l, ids in enumerate(H.levels()):
        ids = [i for i in ids if i != H.root]
        if not ids:
            continue
        a, b = rU[ids], rV[ids]
        print(f"  level {l:2d} nodes {len(ids):4d}  rU mean {a.mean():6.1f} max {a.max():3d}  "
              f"rV mean {b.mean():6.1f} max {b.max():3d}")
    out = torch.empty_like(X)
    for _ in range(2):
        hss.hss_matmul_right(X, H, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        hss.hss_matmul_right(X, H, out=out)
    e1.record()
    torch.cuda.synchronize()
    fl = hss.mult_flops(H, N)
    ms = e0.elapsed_time(e1) / 3
    print(f"  multiply {ms:.2f} ms  flops {fl:.3e}  {fl / ms / 1e9:.1f} TF/s")
