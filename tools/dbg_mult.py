import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1510_04591_b200 as hb
from helpers import config4_system
d, z, rho = config4_system(4096, 4)
sys_ = hb.RankOneSystem(d, z, rho)
sol = hb.solve_secular(sys_)
hb.recompute_weights(sys_.d, sol, sys_.z, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(sys_, sol)
part = hb.build_partition(4096, 128, C.d, C.gamma, C.mu)
print("leaf sizes", sorted(set(hi-lo for lo,hi in part.ranges)), "odd lo", sum(lo % 2 for lo,_ in part.ranges))
r = min(hb.estimate_rank(part, C.d, C.gamma, C.mu, 1e-13), part.min_leaf - 10)
H = hb.rand_hss_construct(C, part, r, p=10, seed=[0, 0])
print("w", r+10, "ws", H.ct.ws, "pmax", H.ct.pmax, "mmax", H.ct.mmax, "r_used", H.r_used)
A = C.to_dense()
dense = hb.hss_to_dense(H)
err = (dense - A).abs()
print("max err", float(err.max()))
# per leaf block rows/cols
for (lo,hi) in part.ranges[:6]:
    print(lo, hi, float(err[:, lo:hi].max()), float(err[lo:hi, :].max()))
# build dense from node views on host
from oracle import hss_oracle as orc
