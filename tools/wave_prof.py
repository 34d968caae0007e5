"""Host/device split of adc_solve: every C-ABI call wrapped in a named Python function so
cProfile attributes host time to it (launch cost for kernels, full cost for host passes).
python tools/wave_prof.py cfg N   (cfg as tools/eigh_prof.py)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200 import _native as nat  # noqa: E402


class _Timed:
    def __init__(self, lib):
        self._lib = lib
        self._cache = {}

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not callable(fn) or not name.startswith("hsseig_"):
            return fn
        if name not in self._cache:
            code = f"def {name}(*a):\n    return fn(*a)\n"
            ns = {"fn": fn}
            exec(code, ns)
            self._cache[name] = ns[name]
        return self._cache[name]


nat._LIB = _Timed(nat.load())
cfg_id, n = sys.argv[1], int(sys.argv[2])
if cfg_id == "1":
    T, cfg = hb.gen_uniform(n, 0), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "2":
    T, cfg = hb.gen_toeplitz(n), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "3":
    T, cfg = hb.gen_kac(n), hb.SolverConfig(rank_eps=1e-13)
else:
    T, cfg = hb.gen_config5(n, 0), hb.SolverConfig(rank_eps=1e-13)
hb.adc_solve(T, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
hb.adc_solve(T, cfg)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0, "cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
pstats.Stats(pr).sort_stats("tottime").print_stats(45)
