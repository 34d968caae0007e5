"""Dense eigenvector update Q @ C (C generated) throughput: python tools/dense_bench.py [k] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else k
d, u, rho = hb.isolated_merge_system(k, 0)
sys_ = hb.RankOneSystem(d, u, rho)
sol = hb.solve_secular(sys_)
hb.recompute_weights(sys_.d, sol, sys_.z, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(sys_, sol)
Q = torch.randn(n, k, dtype=torch.float64, device="cuda")
out = C.right_multiply_into(Q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = C.right_multiply_into(Q, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"k={k} n={n}: {ms:.2f} ms, {2 * n * k * k / ms / 1e9:.1f} TF/s")
ref = Q @ C.to_dense()
print("rel err", float((out - ref).abs().max() / ref.abs().max()))
