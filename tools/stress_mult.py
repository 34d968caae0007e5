"""Repeat the structured multiply on a fixed tree and X; report the first G/F level that differs."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1510_04591_b200 as hb
from paper_1510_04591_b200 import _native as nat
from helpers import config4_system

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
P = int(sys.argv[2]) if len(sys.argv) > 2 else 777
d, z, rho = config4_system(n, 4)
sys_ = hb.RankOneSystem(d, z, rho)
sol = hb.solve_secular(sys_)
hb.recompute_weights(sys_.d, sol, sys_.z, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(sys_, sol)
part = hb.build_partition(n, 128, C.d, C.gamma, C.mu)
r = min(hb.estimate_rank(part, C.d, C.gamma, C.mu, 1e-13), part.min_leaf - 10)
H = hb.rand_hss_construct(C, part, r, p=10, seed=[0, 0])
lib = nat.load()
X = torch.randn(P, n, dtype=torch.float64, device="cuda")
nw = int(lib.hsseig_matmul_work_doubles(P, ctypes.byref(H.ct)))
ws, nl, depth = H.ct.ws, H.ct.n_leaves, H.ct.depth
lvl_total = P * ws * (2 * nl - 2)


def run():
    work = torch.full((nw,), float("nan"), dtype=torch.float64, device="cuda")
    out = torch.full((P, n), float("nan"), dtype=torch.float64, device="cuda")
    nat.check(lib.hsseig_hss_matmul_right(nat.ptr(X), X.stride(0), P, ctypes.byref(H.ct), nat.ptr(out),
                                          out.stride(0), nat.ptr(work), nat.stream_ptr()), "mult")
    torch.cuda.synchronize()
    return work, out


def level(work, base, l):
    off = base + P * ws * ((1 << l) - 2)
    return work[off: off + P * ws * (1 << l)].view(P, (1 << l) * ws)


w0, o0 = run()
print("nan in out", bool(torch.isnan(o0).any()), flush=True)
bad = 0
for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 60):
    w1, o1 = run()
    if torch.equal(o1, o0):
        continue
    bad += 1
    msg = []
    for l in range(depth, 0, -1):
        a, b = level(w1, 0, l), level(w0, 0, l)
        if not torch.equal(a, b):
            e = (a - b).abs()
            rows = torch.nonzero(e.amax(1) > 0).flatten()
            cols = torch.nonzero(e.amax(0) > 0).flatten()
            msg.append(f"G{l} rows {rows[:4].tolist()}..{rows.numel()} cols {cols[:4].tolist()}..{cols.numel()} max {float(e.max()):.2e}")
            break
    for l in range(1, depth + 1):
        a, b = level(w1, lvl_total, l), level(w0, lvl_total, l)
        if not torch.equal(a, b):
            e = (a - b).abs()
            rows = torch.nonzero(e.amax(1) > 0).flatten()
            cols = torch.nonzero(e.amax(0) > 0).flatten()
            msg.append(f"F{l} rows {rows[:4].tolist()}..{rows.numel()} cols {cols[:4].tolist()}..{cols.numel()} max {float(e.max()):.2e}")
            break
    e = (o1 - o0).abs()
    rows = torch.nonzero(e.amax(1) > 0).flatten()
    cols = torch.nonzero(e.amax(0) > 0).flatten()
    msg.append(f"out rows {rows[:4].tolist()}..{rows.numel()} cols {cols[:4].tolist()}..{cols.numel()} max {float(e.max()):.2e}")
    print("it", it, " | ".join(msg), flush=True)
print("bad", bad, flush=True)
