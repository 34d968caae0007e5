"""Device Gaussian draw (csrc/normals.cu) timing + bit-exactness vs NumPy:
python tools/normals_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1510_04591_b200 import sample_rng  # noqa: E402

assert sample_rng.available()
for n in (300_000, 2_752_512, 8_000_000):
    ns = sample_rng.NormalStream(n)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ns.draw([3, 5], n, out)
        ns.fixup()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ns.draw([3, 5], n, out)
    e1.record()
    torch.cuda.synchronize()
    ns.fixup()
    ok = np.array_equal(out.cpu().numpy(), np.random.default_rng([3, 5]).standard_normal(n))
    print(f"n={n}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per draw, exact={ok}")
