"""Host-side timeline of adc_solve per recursion depth (solver.HOST_TRACE marks):
python tools/host_trace.py cfg N   (cfg as tools/eigh_prof.py).  Columns are milliseconds
since the solve began; waits = time the host spent blocked on the device."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200 import solver  # noqa: E402

cfg_id, n = sys.argv[1], int(sys.argv[2])
if cfg_id == "1":
    T, cfg = hb.gen_uniform(n, 0), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "2":
    T, cfg = hb.gen_toeplitz(n), hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
elif cfg_id == "3":
    T, cfg = hb.gen_kac(n), hb.SolverConfig(rank_eps=1e-13)
else:
    T, cfg = hb.gen_config5(n, 0), hb.SolverConfig(rank_eps=1e-13)
if os.environ.get("HSSEIG_METHOD"):
    cfg.method = os.environ["HSSEIG_METHOD"]
for _ in range(2):
    hb.adc_solve(T, cfg)
torch.cuda.synchronize()
solver.HOST_TRACE = []
t0 = time.perf_counter()
hb.adc_solve(T, cfg)
t_ret = time.perf_counter()
torch.cuda.synchronize()
t_end = time.perf_counter()
tr = solver.HOST_TRACE
solver.HOST_TRACE = None
by = {}
for tag, d, t in tr:
    by.setdefault(d, {})[tag] = (t - t0) * 1e3
print(f"returned {1e3 * (t_ret - t0):.2f} ms, device drained {1e3 * (t_end - t0):.2f} ms")
if os.environ.get("HSSEIG_TRACE_SUMMARY"):
    sys.exit(0)
if os.environ.get("HSSEIG_TRACE_FINE"):   # every mark of a depth, as deltas (ms) from the previous one
    seq = {}
    for tag, d, t in tr:
        seq.setdefault(d, []).append((tag, t))
    for d in sorted(seq, reverse=True):
        ev = seq[d]
        print(d, " ".join(f"{b[0]}+{(b[1] - a[1]) * 1e3:.2f}" for a, b in zip(ev, ev[1:])))
    sys.exit(0)
print("depth  begin  rows_wait  deflate  to_queued  roots_wait  to_gather_queued")
for d in sorted(by, reverse=True):
    b = by[d]
    rr = b.get("rows_ready", b["depth_begin"])
    uq = b.get("updates_queued", b["deflated"])
    ro = b.get("roots_ready", uq)
    print(f"{d:5d} {b['depth_begin']:7.2f} {rr - b['depth_begin']:9.2f} {b['deflated'] - rr:8.2f} "
          f"{uq - b['deflated']:9.2f} {ro - uq:10.2f} {b['gather_queued'] - ro:9.2f}")
