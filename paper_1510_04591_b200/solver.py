"""Full divide-and-conquer eigensolver on the GPU (mirror of pkg/src/hsseig/dc.py:174-257).

``adc_solve(T, cfg)`` keeps the reference's recursion (split at n // 2, post-order merge
ids that seed the HSS sample, deflation, dense or HSS update, final ascending order):

* all base cases are solved at once on the device (batched QL, csrc/glue.cu);
* each merge forms z from the last row of Q1 and the first row of Q2 (the only device
  -> host traffic besides eigenvalues), deflates on the host (csrc/glue.cu
  ``hsseig_deflate``), assembles blockdiag(Q1, Q2) in [kept | deflated] column order
  on the device, replays the deflation rotations there, runs the merge body of
  dc.py:236-247 (``dc.merge_update``: secular -> Loewner -> v -> dense or HSS update)
  and gathers the columns into ascending eigenvalue order.

Eigenvalues are returned on the host (NumPy, as the reference); Q stays on the device.
"""
import ctypes
import itertools

import numpy as np
import torch

from . import _native as nat
from .dc import BaseCaseError, EigenResult, MergeRecord, SolverConfig, merge_update
from .flops import FlopCounter

_SQRT2 = np.sqrt(2.0)
MAX_BASE = 32


def _i64(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64), device="cuda")


def _f64(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


def _plan(a, b, base):
    """Leaves of the recursion (dc.py:194-203) and the split-modified diagonal."""
    a = a.copy()
    leaves = []

    def rec(lo, hi):
        if hi - lo <= base:
            leaves.append((lo, hi))
            return
        m = lo + (hi - lo) // 2
        rho = abs(float(b[m - 1]))
        a[m - 1] -= rho          # split (dc.py:82-102): both corner diagonals drop by rho
        a[m] -= rho
        rec(lo, m)
        rec(m, hi)

    rec(0, a.size)
    return a, leaves


def _base_cases(a_mod, b, leaves, stream):
    lib = nat.load()
    sizes = np.array([hi - lo for lo, hi in leaves], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    qoff = np.concatenate([[0], np.cumsum(sizes * sizes)])
    bb = np.concatenate([b[lo:hi - 1] for lo, hi in leaves] + [np.zeros(1)])
    lam = torch.empty(int(off[-1]), dtype=torch.float64, device="cuda")
    Q = torch.empty(int(qoff[-1]), dtype=torch.float64, device="cuda")
    st = torch.zeros(len(leaves), dtype=torch.int32, device="cuda")
    a_d, b_d, off_d, qoff_d = _f64(a_mod), _f64(bb), _i64(off), _i64(qoff)
    nat.check(lib.hsseig_tql2_batched(nat.ptr(a_d), nat.ptr(b_d), nat.ptr(off_d), len(leaves), 30,
                                      nat.ptr(lam), nat.ptr(Q), nat.ptr(qoff_d), nat.ptr(st), stream),
              "tql2_batched")
    bad = st.cpu().numpy()
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise BaseCaseError(f"QL iteration stalled on eigenvalue {int(bad[i]) - 1}")
    lam_h = lam.cpu().numpy()
    out = {}
    for t, (lo, hi) in enumerate(leaves):
        n = hi - lo
        out[(lo, hi)] = (lam_h[off[t]:off[t + 1]].copy(),
                         Q[int(qoff[t]):int(qoff[t]) + n * n].view(n, n))
    return out


def adc_solve(T, cfg=None):
    """Full eigendecomposition of SymTridiagonal T (dc.py:174-191), merges on the GPU."""
    cfg = cfg or SolverConfig()
    if not (np.all(np.isfinite(T.a)) and np.all(np.isfinite(T.b))):
        raise ValueError("matrix has non-finite entries")
    if cfg.base_size > MAX_BASE:
        raise ValueError(f"base_size above {MAX_BASE} is not supported by the device base case")
    nat.require_cuda()
    lib = nat.load()
    s = nat.stream_ptr()
    flops = FlopCounter()
    merges = []
    ids = itertools.count()
    a = np.asarray(T.a, dtype=np.float64)
    b = np.asarray(T.b, dtype=np.float64)
    a_mod, leaves = _plan(a, b, cfg.base_size)
    base = _base_cases(a_mod, b, leaves, s)

    def rec(lo, hi):
        n = hi - lo
        if n <= cfg.base_size:
            return base[(lo, hi)]
        m = lo + (hi - lo) // 2
        n1 = m - lo
        L1, Q1 = rec(lo, m)
        L2, Q2 = rec(m, hi)
        mid = next(ids)
        bk = float(b[m - 1])
        rho = abs(bk)
        theta = 1.0 if bk >= 0.0 else -1.0
        dcat = np.concatenate([L1, L2])
        if rho == 0.0:   # exactly decoupled (dc.py:206-213)
            order = np.argsort(dcat, kind="stable")
            Q = torch.empty(n, n, dtype=torch.float64, device="cuda")
            src = _i64(order)
            nat.check(lib.hsseig_assemble_merge(nat.ptr(Q1), n1, nat.ptr(Q2), n - n1, nat.ptr(src),
                                                nat.ptr(Q), n, s), "assemble")
            return dcat[order], Q
        # merge (dc.py:105-115): z from the boundary rows, joint stable sort
        zrow = torch.cat([Q1[-1], Q2[0]]).cpu().numpy()
        zrow[n1:] *= theta
        z = zrow / _SQRT2
        perm = np.argsort(dcat, kind="stable")
        ds, zs, reff = dcat[perm], z[perm], 2.0 * rho
        # deflation on the host (secular.py:91-156)
        d_out, z_out = np.empty(n), np.empty(n)
        dperm = np.empty(n, dtype=np.int64)
        ri, rj = np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64)
        rc, rs = np.empty(n), np.empty(n)
        nrot = ctypes.c_int64(0)
        P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        k = int(lib.hsseig_deflate(P(ds), P(zs), n, reff, P(d_out), P(z_out), P(dperm), P(ri),
                                   P(rj), P(rc), P(rs), ctypes.byref(nrot), None))
        nr = int(nrot.value)
        rec_ = MergeRecord(size=n, kept=k, n_deflated=n - k)
        merges.append(rec_)
        before = flops.as_dict()
        # W = blockdiag(Q1, Q2) in [kept | deflated] column order, then the rotations
        src = perm[dperm]
        posW = np.empty(n, dtype=np.int64)
        posW[src] = np.arange(n)
        W = torch.empty(n, n, dtype=torch.float64, device="cuda")
        nat.check(lib.hsseig_assemble_merge(nat.ptr(Q1), n1, nat.ptr(Q2), n - n1, nat.ptr(_i64(src)),
                                            nat.ptr(W), n, s), "assemble")
        del Q1, Q2     # the children's blocks are dead once assembled (memory at N = 65536)
        if nr:
            ca, cb = _i64(posW[perm[ri[:nr]]]), _i64(posW[perm[rj[:nr]]])
            cc, ss = _f64(rc[:nr]), _f64(rs[:nr])
            nat.check(lib.hsseig_apply_rotations(nat.ptr(W), n, n, nat.ptr(ca), nat.ptr(cb),
                                                 nat.ptr(cc), nat.ptr(ss), nr, s), "rotations")
        if k > 0:
            lam_k, Qk, _ = merge_update(d_out[:k], z_out[:k], reff, W[:, :k], cfg,
                                        seed=[cfg.seed, mid], flops=flops, record=rec_)
            lam_k = lam_k.cpu().numpy()
        else:
            lam_k, Qk = np.zeros(0), W
        rec_.flops = {p: v - before[p] for p, v in flops.as_dict().items()}
        lam_cat = np.concatenate([lam_k, d_out[k:]])
        order = np.argsort(lam_cat, kind="stable")
        if k == 0:
            return lam_cat[order], W[:, torch.as_tensor(order, device="cuda")].contiguous()
        # gather into W's own storage: the deflated columns move to a compact copy first
        Wd = W[:, k:].contiguous() if k < n else Qk
        nat.check(lib.hsseig_gather_columns(nat.ptr(Qk), Qk.stride(0), ctypes.c_void_p(Wd.data_ptr() - 8 * k),
                                            max(n - k, 1), k, nat.ptr(_i64(order)), n, n, nat.ptr(W),
                                            n, s), "gather")
        del Wd, Qk
        return lam_cat[order], W

    lam, Q = rec(0, T.n)
    return EigenResult(lam=lam, Q=Q, merges=merges, flops=flops)
