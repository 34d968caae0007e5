"""Sample products against cuBLAS on the dense C (checker): python tools/check_sample.py [k]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200.hss import draw_omega  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d, u, rho = hb.isolated_merge_system(k, 0)
s = hb.RankOneSystem(d, u, rho)
sol = hb.solve_secular(s)
hb.recompute_weights(d, sol, u, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(s, sol)
w = 82
om = draw_omega(k, w, [0, 0])
Y, Z = C.sample(om)
ey = ez = 0.0
for r0 in range(0, k, 4096):
    blk = C.block(range(r0, min(k, r0 + 4096)), range(k))
    Yr = blk @ om
    ey = max(ey, float((Y[r0:r0 + 4096] - Yr).abs().max() / Yr.abs().max()))
    if r0 == 0:
        Zr = blk.T @ om[r0:r0 + 4096]
    else:
        Zr += blk.T @ om[r0:r0 + 4096]
ez = float((Z - Zr).abs().max() / Zr.abs().max())
print(f"k={k} sample rel err Y {ey:.3e} Z {ez:.3e}")
