"""Per-phase cycle split of the ID elimination (block 0 of every id_kernel launch) on the
config-4 tree: rebuild with HSSEIG_NVCC_EXTRA=-DHSSEIG_ID_TIMING, then
python tools/id_timing.py [N]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200 import _native as nat  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = nat.load()
d, u, rho = hb.isolated_merge_system(N, 0)
s = hb.RankOneSystem(d, u, rho)
sol = hb.solve_secular(s)
hb.recompute_weights(d, sol, u, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(s, sol)
part = hb.build_partition(N, 128, C.d, C.gamma, C.mu)
r = min(hb.estimate_rank(part, C.d, C.gamma, C.mu, 1e-13, 100), part.min_leaf - 10)
hb.rand_hss_construct(C, part, r, p=10, seed=[0, 0])
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
lib.hsseig_debug_id_timing(out, 1)
hb.rand_hss_construct(C, part, r, p=10, seed=[0, 0])
torch.cuda.synchronize()
lib.hsseig_debug_id_timing(out, 0)
v = list(out)
steps = max(v[4], 1)
names = ["warp-0 pivot + reflector", "reflector barrier wait", "own update", "end-of-step wait"]
print(f"steps {v[4]}  elimination {v[5]} cyc  finish {v[6]} cyc  (block 0 of 8 launches)")
for i, nm in enumerate(names):
    print(f"  {nm:28s} {v[i] / steps:8.0f} cyc/step  ({100 * v[i] / max(v[5], 1):4.1f}% of elimination)")
