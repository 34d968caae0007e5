"""One ADC1 (SRRSC) construction of a config-2-sized top merge, for timing / ncu:
python tools/srrsc_prof.py [k] [leaf] [reps].  The rank-one system is the Toeplitz top merge
(poles: the two halves' eigenvalues interleaved, mirror halves deflated away)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
h = k // 2
d = np.sort(np.concatenate([2 + 2 * np.cos(np.arange(1, h + 1) * np.pi / (h + 1)),
                            2 + 2 * np.cos(np.arange(1, k - h + 1) * np.pi / (k - h + 1)) + 1e-4]))
u = np.random.default_rng(0).standard_normal(k)
u /= np.linalg.norm(u)
sys_ = hb.RankOneSystem(d, u, 1.0)
sol = hb.solve_secular(sys_)
hb.recompute_weights(sys_.d, sol, sys_.z, rho=1.0)
C = hb.CauchyEvecMatrix.from_secular(sys_, sol)
part = hb.build_partition(k, leaf, C.d, C.gamma, C.mu)
cap = hb.srrsc_cap(part)
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = hb.srrsc_hss_construct(C, part, cap)
    torch.cuda.synchronize()
    print(f"k={k} leaves={part.n_leaves} cap={cap} r_used={H.r_used} flagged={H.flagged} "
          f"construct {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
