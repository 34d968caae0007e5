"""e2e (streamed host I/O) config-4 merge time per step: python tools/e2e_probe.py [N] [chunks]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200.merge_pipeline import MergePipeline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 16
d, u, rho = hb.isolated_merge_system(n, 0)
cfg = hb.SolverConfig(leaf_size=128, hss_threshold=512, rank_eps=1e-13)
pipe = MergePipeline(n, cfg, rows=n)
hQ = torch.randn(n, n, dtype=torch.float64).pin_memory()
hOut = torch.empty_like(hQ).pin_memory()
hd, hu = torch.as_tensor(d).pin_memory(), torch.as_tensor(u).pin_memory()
X = torch.empty(n, n, dtype=torch.float64, device="cuda")
out = torch.empty_like(X)
for it in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dd, du = hd.to("cuda", non_blocking=True), hu.to("cuda", non_blocking=True)
    info = pipe.run(dd, du, rho, X, seed=[0, 0], out=out, host_io=(hQ, hOut), chunks=chunks)
    e1.record()
    torch.cuda.synchronize()
    print(chunks, it, f"e2e {e0.elapsed_time(e1):.1f} ms",
          {k: round(v, 2) for k, v in info["ms"].items()}, flush=True)
