"""Dump the GPU sample (Y, Z) of the config-4 system at n for offline error analysis."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402
from oracle import hss_oracle as orc  # noqa: E402
n = int(sys.argv[1])
d, u, rho = hb.isolated_merge_system(n, 0)
G, _, _ = orc.generators_from_roots(d, u, rho)
C = hb.CauchyEvecMatrix(G.d, G.gam, G.mu, G.zh, G.v)
ranges = orc.leaf_ranges(n, 128, G.mu)
r = min(orc.rank_estimate(ranges, G.d, G.gam, G.mu, 1e-13), min(h - l for l, h in ranges) - 10)
Om = orc.sample_block(n, r + 10, [0, 0])
Y, Z = C.sample(torch.as_tensor(Om, device="cuda"))
np.savez(f"gpurun_out/c4_yz_{n}.npz", Y=Y.cpu().numpy(), Z=Z.cpu().numpy())
