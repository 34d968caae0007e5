"""Secular kernel timing at config-4 size: python tools/sec_bench.py [k]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d, u, rho = hb.isolated_merge_system(k, 0)
sys_ = hb.RankOneSystem(d, u, rho)
for _ in range(2):
    hb.solve_secular(sys_)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sol = hb.solve_secular(sys_, check=False)
e1.record()
torch.cuda.synchronize()
hb.secular.finish_secular(sol, k)
print(os.environ.get("HSSEIG_SEC_VARIANT", "0"), "secular ms", e0.elapsed_time(e1) / 5, "iters", sol.iterations)
