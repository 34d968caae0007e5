"""Latency of the shared-memory interpolative decomposition (the construction's ID) on
sample-like matrices: python tools/id_bench.py.  A p x w block of a numerically rank-r
matrix plus noise at 1e-16 (what the upper tree levels factor), batch 1 and batch 512."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1510_04591_b200 import _native as nat  # noqa: E402

lib = nat.load()
for p, w, batch in ((168, 84, 1), (168, 84, 4), (128, 84, 512)):
    rng = np.random.default_rng(0)
    r = 70
    M = np.stack([rng.standard_normal((p, r)) @ rng.standard_normal((r, w)) * np.exp(-np.arange(w) / 4)
                  + 1e-16 * rng.standard_normal((p, w)) for _ in range(batch)])
    Md = torch.as_tensor(M, device="cuda")
    X = torch.zeros(batch, p, w, dtype=torch.float64, device="cuda")
    J = torch.zeros(batch, w, dtype=torch.int32, device="cuda")
    rk = torch.zeros(batch, dtype=torch.int32, device="cuda")
    rs = torch.zeros(batch, dtype=torch.float64, device="cuda")
    sat = torch.zeros(batch, dtype=torch.int32, device="cuda")

    def run():
        nat.check(lib.hsseig_interp_decomp(nat.ptr(Md), w, p * w, p, w, batch, 1e-15, w,
                                           nat.ptr(X), w, p * w, nat.ptr(J), nat.ptr(rk),
                                           nat.ptr(rs), nat.ptr(sat), nat.stream_ptr()), "id")
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"p={p} w={w} batch={batch}: {1e3 * e0.elapsed_time(e1) / 10:.1f} us per launch, "
          f"rank {int(rk[0])}", flush=True)
