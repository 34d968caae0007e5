"""One (or more) isolated merges at size n for profiling: python tools/prof_merge.py N [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200.merge_pipeline import MergePipeline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, u, rho = hb.isolated_merge_system(n, 0)
X = torch.randn(n, n, dtype=torch.float64, device="cuda") / n ** 0.5
cfg = hb.SolverConfig(leaf_size=128, hss_threshold=512, rank_eps=1e-13)
pipe = MergePipeline(n, cfg, rows=n)
dd, du = torch.as_tensor(d, device="cuda"), torch.as_tensor(u, device="cuda")
out = torch.empty_like(X)
for i in range(reps):
    info = pipe.run(dd, du, rho, X, seed=[0, 0], out=out)
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in info["ms"].items()}, info["r_used"], info["used_hss"])
