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
import os

import numpy as np
import torch

from . import _native as nat
from .cauchy import DENSE_PANEL_BYTES, DENSE_PANEL_MIN_K, CauchyEvecMatrix
from .dc import (HSS_METHODS, BaseCaseError, EigenResult, HssJob, MergeRecord, SolverConfig,
                 merge_update, update_vectors_hss_many)
from .flops import FlopCounter, cauchy_eval_flops, gemm_flops, secular_flops
from .secular import SecularConvergenceError, WeightRecomputationError

_SQRT2 = np.sqrt(2.0)
MAX_BASE = 160   # largest device base case (csrc/glue.cu kQLBig)

# When a list, solve_subtree appends one (kind, start event, end event, algorithmic bytes)
# per recursion depth for the HBM-bound glue kernels (bench.py's glue GB/s line):
#   "assemble": blockdiag(Q1, Q2) columns into W (child entries read, W written) + the
#               Givens replay (two columns read and written per rotation and row);
#   "gather":   the final column order (the n x n block read and written).
GLUE_PROFILE = None


DENSE_STREAMS = int(os.environ.get("HSSEIG_DENSE_STREAMS", "4"))   # panel updates of a depth in flight
HOST_TRACE = None   # set to a list: (tag, depth, perf_counter) marks of solve_subtree's host side


def _mark(tag, depth):
    if HOST_TRACE is not None:
        import time
        HOST_TRACE.append((tag, depth, time.perf_counter()))


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


class _Pack:
    """Host arrays packed into one pinned staging buffer and sent with ONE host->device
    copy (a level of the wave schedule uploads ~20 small index arrays; one pageable
    upload each cost ~70 us of host time at config 5).  The device views keep the
    buffer alive until the launches reading them are queued."""
    _T = {np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64,
          np.dtype(np.int32): torch.int32}

    def __init__(self):
        self.parts = []

    def add(self, x, dtype=np.int64):
        self.parts.append(np.ascontiguousarray(x, dtype=dtype).reshape(-1))
        return self

    def send(self):
        offs, o = [], 0
        for p in self.parts:
            offs.append(o)
            o += max(16, (p.nbytes + 15) & ~15)
        host = torch.empty(o, dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for p, q in zip(self.parts, offs):
            hv[q:q + p.nbytes] = p.view(np.uint8)
        dev = host.to("cuda", non_blocking=True)
        # one reinterpretation of the staging buffer per element type; a part is then a slice
        typed = {}
        out = []
        for p, q in zip(self.parts, offs):
            t = typed.get(p.dtype)
            if t is None:
                t = typed[p.dtype] = dev.view(self._T[p.dtype])
            e = q // p.itemsize
            out.append(t[e:e + max(p.size, 1)])
        return out


def _base_cases_flat(a_mod, b, lo, hi, stream):
    """Every leaf (rows [lo[t], hi[t]), contiguous and ascending) solved in one launch
    (batched QL, csrc/glue.cu).  Returns (eigenvalues of all leaves on the host in row
    order, Q buffer on the device, qoff): leaf t's Q is Q[qoff[t]:qoff[t+1]] (n x n)."""
    lib = nat.load()
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    sizes = hi - lo
    if sizes.size and int(sizes.max()) > MAX_BASE:
        raise ValueError(f"base case of order {int(sizes.max())} above the device QL's {MAX_BASE}")
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    qoff = np.concatenate([[0], np.cumsum(sizes * sizes)]).astype(np.int64)
    L0, L1 = int(lo[0]), int(hi[-1])
    # off-diagonals of every leaf: drop the couplings b[hi - 1] between neighbours
    bb = np.concatenate([np.delete(b[L0:L1 - 1], hi[:-1] - 1 - L0), [0.0]])
    a_d, b_d, off_d, qoff_d = (_Pack().add(a_mod[L0:L1], np.float64).add(bb, np.float64)
                               .add(off).add(qoff).send())
    lam = torch.empty(int(off[-1]), dtype=torch.float64, device="cuda")
    Q = torch.empty(int(qoff[-1]), dtype=torch.float64, device="cuda")
    st = torch.zeros(len(lo), dtype=torch.int32, device="cuda")
    nat.check(lib.hsseig_tql2_batched(nat.ptr(a_d), nat.ptr(b_d), nat.ptr(off_d), len(lo),
                                      int(sizes.max()), 30, nat.ptr(lam), nat.ptr(Q),
                                      nat.ptr(qoff_d), nat.ptr(st), 0, stream),
              "tql2_batched")
    bad = st.cpu().numpy()
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise BaseCaseError(f"QL iteration stalled on eigenvalue {int(bad[i]) - 1}")
    return lam.cpu().numpy(), Q, qoff


def _base_cases(a_mod, b, leaves, stream):
    lo = np.array([l for l, _ in leaves], dtype=np.int64)
    hi = np.array([h for _, h in leaves], dtype=np.int64)
    lam_h, Q, qoff = _base_cases_flat(a_mod, b, lo, hi, stream)
    out = {}
    for t, (l, h) in enumerate(leaves):
        n = h - l
        out[(l, h)] = (lam_h[l - lo[0]:h - lo[0]].copy(),
                       Q[int(qoff[t]):int(qoff[t]) + n * n].view(n, n))
    return out


def adc_solve_recursive(T, cfg=None):
    """Full eigendecomposition of SymTridiagonal T (dc.py:174-191), one merge at a time."""
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


# ----------------------------------------------------------------------------------------
# Level-batched schedule: every merge of one recursion depth runs in one set of launches.
# ----------------------------------------------------------------------------------------
class _Tree:
    """Recursion nodes (dc.py:194-203: split at n // 2, merge ids in postorder) as arrays in
    postorder, built level by level with NumPy (a Python recursion over the 8191 nodes of
    config 5 cost 12 ms of host time before the first launch).  A subtree is the contiguous
    id range [i - size[i] + 1, i].  Indexing or iterating yields per-node dicts with the keys
    lo, hi, depth, leaf and, for merges, left, right, split, mid."""

    def __init__(self, n, base):
        lo, hi = np.zeros(1, np.int64), np.full(1, n, np.int64)
        levels = []
        while len(lo):
            inner = (hi - lo) > base
            m = lo + (hi - lo) // 2
            levels.append((lo, hi, inner, m))
            li, hi_i, mi = lo[inner], hi[inner], m[inner]
            lo = np.stack([li, mi], 1).reshape(-1)
            hi = np.stack([mi, hi_i], 1).reshape(-1)
        # subtree sizes bottom-up; the children of a level's j-th merge are nodes 2j, 2j+1 below
        sizes = [None] * len(levels)
        for d in range(len(levels) - 1, -1, -1):
            inner = levels[d][2]
            sz = np.ones(len(inner), np.int64)
            if inner.any():
                c = sizes[d + 1]
                sz[inner] += c[0::2] + c[1::2]
            sizes[d] = sz
        total = int(sizes[0][0])
        self.lo, self.hi, self.depth, self.split, self.left, self.right, self.size = (
            np.zeros(total, np.int64) for _ in range(7))
        self.leaf = np.ones(total, bool)
        post = np.array([total - 1], np.int64)
        for d, (lo, hi, inner, m) in enumerate(levels):
            self.lo[post], self.hi[post], self.depth[post], self.size[post] = lo, hi, d, sizes[d]
            if not inner.any():
                break
            pi = post[inner]
            right = pi - 1
            left = right - sizes[d + 1][1::2]
            self.leaf[pi] = False
            self.split[pi], self.left[pi], self.right[pi] = m[inner], left, right
            post = np.stack([left, right], 1).reshape(-1)
        self.mid = np.cumsum(~self.leaf) - 1

    def __len__(self):
        return len(self.lo)

    def __getitem__(self, i):
        i = int(i)
        nd = {"lo": int(self.lo[i]), "hi": int(self.hi[i]), "depth": int(self.depth[i]),
              "leaf": bool(self.leaf[i])}
        if not nd["leaf"]:
            nd.update(left=int(self.left[i]), right=int(self.right[i]), split=int(self.split[i]),
                      mid=int(self.mid[i]))
        return nd

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def split_diagonal(self, a, b, max_depth=None):
        """The diagonal with the split modifications (dc.py:82-102) of every merge (above
        max_depth): both corner diagonals drop by rho = |b[m-1]|.  Blocks hold >= 2 rows, so
        no entry is touched by two splits and the update order is immaterial."""
        a = np.array(a, dtype=np.float64)
        sel = ~self.leaf if max_depth is None else (~self.leaf & (self.depth < max_depth))
        m = self.split[sel]
        rho = np.abs(b[m - 1])
        a[m - 1] -= rho
        a[m] -= rho
        return a


def _tree(n, base):
    nodes = _Tree(n, base)
    return nodes, len(nodes) - 1


def _u64(ptrs):
    return torch.as_tensor(np.asarray(ptrs, dtype=np.uint64).view(np.int64), device="cuda")


def _i32(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32), device="cuda")


def _cptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def adc_solve(T, cfg=None):
    """Full eigendecomposition of SymTridiagonal T (dc.py:174-257), level-batched on the GPU.

    The recursion, split, deflation, merge ids (HSS sample seeds) and merge records are
    the reference's.  All merges of one depth share their launches: boundary rows ->
    host deflation (one C call) -> assembly + Givens replay -> segmented secular /
    Loewner / normalizers -> grouped dense updates (HSS merges individually) -> final
    column order.  Two host synchronisations per depth.
    """
    cfg = cfg or SolverConfig()
    if not (np.all(np.isfinite(T.a)) and np.all(np.isfinite(T.b))):
        raise ValueError("matrix has non-finite entries")
    if cfg.base_size > MAX_BASE:
        raise ValueError(f"base_size above {MAX_BASE} is not supported by the device base case")
    nat.require_cuda()
    a = np.asarray(T.a, dtype=np.float64)
    b = np.asarray(T.b, dtype=np.float64)
    nodes, root = _tree(T.n, cfg.base_size)
    a_mod = nodes.split_diagonal(a, b) if cfg.base_size >= 3 else _plan(a, b, cfg.base_size)[0]
    lam, Q, records = solve_subtree(a_mod, b, nodes, root, cfg)
    flops = FlopCounter()
    merges = [records[k] for k in sorted(records)]
    for p_ in FlopCounter.PHASES:
        setattr(flops, p_, getattr(flops, p_) + sum(r.flops.get(p_, 0) for r in merges))
    return EigenResult(lam=lam, Q=Q, merges=merges, flops=flops)


def solve_subtree(a_mod, b, nodes, sub, cfg):
    """Eigenpairs of the recursion node `sub` (its base cases and every merge below it,
    level-batched); a_mod carries all split modifications (_plan).  Returns (lam host,
    Q device n x n in the node's local coordinates, {merge id: MergeRecord})."""
    lib = nat.load()
    s = nat.stream_ptr()
    f64 = dict(dtype=torch.float64, device="cuda")
    # nodes are in postorder, so the subtree is the id range [leftmost leaf, sub]
    first = int(sub - nodes.size[sub] + 1)
    rng = slice(first, sub + 1)
    lo_a, hi_a, dep_a, leaf_a = nodes.lo[rng], nodes.hi[rng], nodes.depth[rng], nodes.leaf[rng]
    split_a, mid_a = nodes.split[rng], nodes.mid[rng]
    left_a = np.where(leaf_a, 0, nodes.left[rng] - first)
    right_a = np.where(leaf_a, 0, nodes.right[rng] - first)
    ntab = len(lo_a)
    base_lo = int(lo_a[-1])
    leaf_idx = np.flatnonzero(leaf_a)        # postorder visits the leaves left to right
    lam_all, Qbase, lqoff = _base_cases_flat(a_mod, b, lo_a[leaf_idx], hi_a[leaf_idx], s)
    # boundary rows (the z of dc.py:112) of every finished block on the host, by node: the
    # leaves' from the base cases here, a merge's from the early row gather of its depth,
    # so the next depth's deflation runs while the device is still gathering
    nl = hi_a[leaf_idx] - lo_a[leaf_idx]
    rows_h = np.zeros(0)
    if len(leaf_idx):
        first_i = np.repeat(lqoff[:-1], nl) + (np.arange(int(nl.sum())) - np.repeat(np.cumsum(nl) - nl, nl))
        last_i = first_i + np.repeat((nl - 1) * nl, nl)
        rows_h = Qbase[torch.as_tensor(np.concatenate([first_i, last_i]), device="cuda")].cpu().numpy()
    lrow0 = np.concatenate([[0], np.cumsum(nl)]).astype(np.int64)
    # offsets of every node's first / last row in [leaf rows | the last depth's row gather]
    first_off = np.zeros(ntab, dtype=np.int64)
    last_off = np.zeros(ntab, dtype=np.int64)
    first_off[leaf_idx] = lrow0[:-1]
    last_off[leaf_idx] = int(lrow0[-1]) + lrow0[:-1]
    is_left = np.zeros(ntab, dtype=bool)
    has_parent = np.zeros(ntab, dtype=bool)
    inner_j = np.flatnonzero(~leaf_a)
    is_left[left_a[inner_j]] = True
    has_parent[left_a[inner_j]] = has_parent[right_a[inner_j]] = True
    pending = None      # (event, pinned rows) of the last depth's early row gather
    pending_records = []
    # per node: device address of its Q block (row-major n x n) and the buffer holding it
    qptr = np.zeros(ntab, dtype=np.uint64)
    qptr[leaf_idx] = np.uint64(Qbase.data_ptr()) + (8 * lqoff[:-1]).astype(np.uint64)
    live = {}
    records = {}
    bm = ctypes.c_int32(0)
    bn = ctypes.c_int32(0)
    lib.hsseig_wave_tile_shape(ctypes.byref(bm), ctypes.byref(bn))
    bm, bn = bm.value, bn.value
    internal = np.flatnonzero(~leaf_a)
    top = int(dep_a[-1])
    for depth in range(int(dep_a.max()) - 1, top - 1, -1):
        ms = internal[dep_a[internal] == depth]
        if not len(ms):
            continue
        nm = len(ms)
        lo_m, sp_m = lo_a[ms], split_a[ms]
        n1 = sp_m - lo_m
        n2 = hi_a[ms] - sp_m
        nv = n1 + n2
        roff = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
        nrows = int(roff[-1])
        rm = np.repeat(np.arange(nm, dtype=np.int32), nv)      # row -> merge (device table)
        # the merges of a depth cover increasing disjoint index ranges; one contiguous range
        # when the depth holds no leaf (a slice instead of a 65536-entry index array)
        if nm == 1 or np.array_equal(lo_m[1:], hi_a[ms[:-1]]):
            rows = slice(int(lo_m[0] - base_lo), int(lo_m[0] - base_lo) + nrows)
        else:
            rows = np.arange(nrows) + np.repeat(lo_m - base_lo - roff[:-1], nv)
        L = np.ascontiguousarray(lam_all[rows])
        q1, q2, n1_d, n2_d, nv_d, roff_d = (
            _Pack().add(qptr[left_a[ms]].view(np.int64)).add(qptr[right_a[ms]].view(np.int64))
            .add(n1).add(n2).add(nv).add(roff).send())
        # boundary rows of the children (sync 1: the early row gather of the previous depth)
        src_rows = rows_h
        _mark("depth_begin", depth)
        if pending is not None:
            ev_rows, rows_pin = pending
            ev_rows.synchronize()
            _mark("rows_ready", depth)
            src_rows = np.concatenate([rows_h, rows_pin.numpy()])
            pending = None
        # z rows: [last row of the left child | first row of the right child] per merge
        st_z = np.stack([last_off[left_a[ms]], first_off[right_a[ms]]], 1).reshape(-1)
        ln_z = np.stack([n1, n2], 1).reshape(-1)
        z_at = np.cumsum(ln_z) - ln_z
        if np.array_equal(st_z - st_z[0], z_at):
            # every child is a merge of the previous depth: its row gather is already laid
            # out as [last row of the left child | first row of the right child] per merge
            zrow = np.ascontiguousarray(src_rows[int(st_z[0]):int(st_z[0]) + nrows])
        else:
            zrow = src_rows[np.repeat(st_z - z_at, ln_z) + np.arange(nrows)]
        bk = np.ascontiguousarray(b[sp_m - 1], dtype=np.float64)
        kept = np.empty(nm, dtype=np.int64)
        rho_eff = np.empty(nm)
        d_out, z_out = np.empty(nrows), np.empty(nrows)
        src = np.empty(nrows, dtype=np.int64)
        rot_off = np.empty(nm + 1, dtype=np.int64)
        ca, cb = np.empty(nrows, dtype=np.int64), np.empty(nrows, dtype=np.int64)
        rc, rs = np.empty(nrows), np.empty(nrows)
        ktot = int(lib.hsseig_wave_deflate(nm, _cptr(n1), _cptr(n2), _cptr(roff), _cptr(L),
                                           _cptr(zrow), _cptr(bk), _cptr(kept), _cptr(rho_eff),
                                           _cptr(d_out), _cptr(z_out), _cptr(src), _cptr(rot_off),
                                           _cptr(ca), _cptr(cb), _cptr(rc), _cptr(rs)))
        _mark("deflated", depth)
        # W_m holds only the kept columns and the deflated columns a rotation touches (the
        # other deflated columns are plain child eigenvectors, read by the final gather);
        # rows padded to an even leading dimension for the TMA engine
        wd = np.empty(nm, dtype=np.int64)
        coff = np.empty(nm + 1, dtype=np.int64)
        csrc = np.empty(nrows, dtype=np.int64)
        cmap = np.empty(nrows, dtype=np.int64)
        lib.hsseig_wave_compact(nm, _cptr(roff), _cptr(kept), _cptr(src), _cptr(rot_off), _cptr(ca),
                                _cptr(cb), _cptr(wd), _cptr(coff), _cptr(csrc), _cptr(cmap))
        ldw = wd + (wd & 1)
        woff = np.concatenate([[0], np.cumsum(nv * ldw)]).astype(np.int64)
        ooff = np.concatenate([[0], np.cumsum(nv * nv)]).astype(np.int64)
        nrot = int(rot_off[-1])
        # the kept rank-one systems, concatenated
        segs = np.flatnonzero(kept > 0)
        nseg = len(segs)
        ks = kept[segs]
        koff = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
        kidx = np.repeat(roff[segs] - koff[:-1], ks) + np.arange(ktot)
        qoff = np.concatenate([[0], np.cumsum(nv * kept)]).astype(np.int64)
        # update route of every system: HSS (adc-rand / adc-srrsc above the threshold), a materialised
        # C panel on the TMA/DMMA engine (k >= DENSE_PANEL_MIN_K) or the grouped dense tiles
        nvs = nv[segs]
        hss_q = (ks > cfg.hss_threshold) if cfg.method in HSS_METHODS else np.zeros(nseg, bool)
        big_q = ~hss_q & (ks >= DENSE_PANEL_MIN_K)
        small = np.flatnonzero(~hss_q & ~big_q)
        # K order of every panel update, [child 1 only | rotated | child 2 only] (the rows of
        # blockdiag(Q1, Q2) above / below the split see only their own child's kept columns
        # and the ones a deflation rotation mixed: hsseig_dense_update_halves)
        big = np.flatnonzero(big_q)
        # ... also for the HSS merges wide enough for the panel path, whose flagged trees fall
        # back to the dense update (the classification rides along; the panel loop below
        # takes the first len(big) entries)
        hss_p = np.flatnonzero(hss_q & (ks >= DENSE_PANEL_MIN_K))
        nbig = len(big)
        big = np.concatenate([big, hss_p])
        kperm, ka_b, kb_b = np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
        boff = np.zeros(1, np.int64)
        if len(big):
            mb, kb_ = segs[big], ks[big]
            boff = np.concatenate([[0], np.cumsum(kb_)]).astype(np.int64)
            seg_b = np.repeat(np.arange(len(big)), kb_)
            pos_b = np.arange(int(boff[-1])) - boff[seg_b]
            cls = np.where(src[roff[mb][seg_b] + pos_b] < n1[mb][seg_b], 0, 2)
            nr_b = rot_off[mb + 1] - rot_off[mb]
            if nr_b.sum():
                seg_r = np.repeat(np.arange(len(big)), nr_b)
                ridx = np.repeat(rot_off[mb] - (np.cumsum(nr_b) - nr_b), nr_b) + np.arange(int(nr_b.sum()))
                for cc in (ca[ridx], cb[ridx]):
                    ok = cc < kb_[seg_r]
                    cls[boff[seg_r[ok]] + cc[ok]] = 1
            kperm = np.lexsort((cls, seg_b)) - boff[seg_b]       # stable within a merge
            ka_b = np.add.reduceat((cls <= 1).astype(np.int64), boff[:-1])
            kb_b = np.add.reduceat((cls == 0).astype(np.int64), boff[:-1])
        # K orders of the HSS merges (host side, handed to their jobs), then the panel merges alone
        hss_halves = {int(q): (kperm[boff[nbig + i]:boff[nbig + i + 1]], int(ka_b[nbig + i]), int(kb_b[nbig + i]))
                      for i, q in enumerate(hss_p.tolist())}
        big, kperm, ka_b, kb_b = big[:nbig], kperm[:boff[nbig]], ka_b[:nbig], kb_b[:nbig]
        mt, nt = -(-nvs[small] // bm), -(-ks[small] // bn)
        cnt = mt * nt
        tk = np.empty((int(cnt.sum()), 3), dtype=np.int32)
        if len(tk):
            tq = np.repeat(np.arange(len(small)), cnt)
            loc = np.arange(len(tk)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            tk[:, 0] = small[tq]
            tk[:, 1] = loc // nt[tq]
            tk[:, 2] = loc % nt[tq]
        # rotation runs (one survivor each; disjoint columns): the rotate kernel's tasks
        if nrot:
            ca_h = ca[:nrot]
            starts = np.ones(nrot, dtype=bool)
            starts[1:] = ca_h[1:] != ca_h[:-1]
            starts[rot_off[:-1][np.diff(rot_off) > 0]] = True     # merge boundaries
            run_t = np.flatnonzero(starts)
            run_off = np.searchsorted(run_t, rot_off).astype(np.int64)
            run_t = np.append(run_t, nrot)
            rot_tasks = int((nv * np.diff(run_off)).max())
        else:
            run_t, run_off, rot_tasks = np.zeros(1, np.int64), np.zeros(nm + 1, np.int64), 0
        st0 = np.zeros((nseg, 8), dtype=np.int64)
        st0[:, 1:4] = ks[:, None]
        _mark("t_indexed", depth)
        (woff_d, wd_d, row_merge, csrc_d, coff_d, rot_d1, rot_d2, rot_d3, rot_d4, dk, zk,
         koff_d, seg_of, rho_d, st, t_woff, t_nv, t_qoff, t_tk, t_ldw, run_t_d, run_off_d,
         kperm_d) = (
            _Pack().add(woff).add(wd).add(rm, np.int32).add(csrc[:int(coff[-1])]).add(coff)
            .add(ca[:nrot]).add(cb[:nrot]).add(rc[:nrot], np.float64)
            .add(rs[:nrot], np.float64).add(d_out[kidx], np.float64).add(z_out[kidx], np.float64)
            .add(koff).add(np.repeat(np.arange(nseg, dtype=np.int32), ks), np.int32)
            .add(rho_eff[segs], np.float64).add(st0).add(woff[segs]).add(nvs).add(qoff[segs])
            .add(tk, np.int32).add(ldw[segs]).add(run_t).add(run_off).add(kperm).send())
        _mark("t_packed", depth)
        W = torch.empty(max(int(woff[-1]), 2), **f64)
        prof = GLUE_PROFILE
        if prof is not None:
            cm = np.repeat(np.arange(nm), np.diff(coff))
            src_rows = np.where(csrc[:int(coff[-1])] < n1[cm], n1[cm], n2[cm])
            rot_rows = np.repeat(nv, np.diff(rot_off))
            gbytes = 8 * (int((nv * wd).sum()) + int(src_rows.sum())) + 32 * int(rot_rows.sum())
            ev_g = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev_g[0].record()
        nat.check(lib.hsseig_wave_assemble(nat.ptr(q1), nat.ptr(q2), nat.ptr(n1_d), nat.ptr(n2_d),
                                           nat.ptr(roff_d), nat.ptr(row_merge), nat.ptr(csrc_d),
                                           nat.ptr(coff_d), nat.ptr(wd_d), nat.ptr(W), nat.ptr(woff_d),
                                           nrows, s), "wave_assemble")
        if nrot:
            nat.check(lib.hsseig_wave_rotate(nat.ptr(W), nat.ptr(woff_d), nat.ptr(nv_d), nat.ptr(wd_d),
                                             nat.ptr(run_t_d), nat.ptr(run_off_d), nat.ptr(rot_d1),
                                             nat.ptr(rot_d2), nat.ptr(rot_d3), nat.ptr(rot_d4), nm,
                                             rot_tasks, s),
                      "wave_rotate")
        if prof is not None:
            ev_g[1].record()
            prof.append(("assemble", ev_g[0], ev_g[1], gbytes))
        _mark("t_assembled", depth)
        Qk = torch.empty(max(int(qoff[-1]), 1), **f64)
        hss_m = set(np.flatnonzero(hss_q).tolist())
        seg_iters = np.zeros(nseg, dtype=np.int64)
        if nseg:
            lam_k, gam, mu, dn, zh, vv = (torch.empty(ktot, **f64) for _ in range(6))
            its = torch.empty(ktot, dtype=torch.int32, device="cuda")
            work = torch.empty(ktot + nseg, **f64)
            nat.check(lib.hsseig_wave_secular(nat.ptr(dk), nat.ptr(zk), nat.ptr(koff_d), nat.ptr(seg_of),
                                              nat.ptr(rho_d), nseg, ktot, nat.ptr(lam_k), nat.ptr(gam),
                                              nat.ptr(mu), nat.ptr(its), nat.ptr(work), nat.ptr(st), s),
                      "wave_secular")
            nat.check(lib.hsseig_wave_dnext(nat.ptr(dk), nat.ptr(gam), nat.ptr(mu), nat.ptr(koff_d),
                                            nat.ptr(seg_of), ktot, nat.ptr(dn), s), "wave_dnext")
            nat.check(lib.hsseig_wave_loewner(nat.ptr(dk), nat.ptr(dn), nat.ptr(gam), nat.ptr(mu),
                                              nat.ptr(zk), nat.ptr(koff_d), nat.ptr(seg_of),
                                              nat.ptr(rho_d), ktot, nat.ptr(zh), nat.ptr(st), s),
                      "wave_loewner")
            nat.check(lib.hsseig_wave_normalizers(nat.ptr(dk), nat.ptr(dn), nat.ptr(gam), nat.ptr(mu),
                                                  nat.ptr(zh), nat.ptr(koff_d), nat.ptr(seg_of), ktot,
                                                  nat.ptr(vv), s), "wave_normalizers")
            # statuses and roots (sync 2) go to pinned host buffers right behind the secular
            # stage; the dense updates are queued before the host waits, so the host-side
            # checks, HSS set-up and final ordering below overlap them on the device
            _mark("t_secular", depth)
            st_pin = torch.empty((nseg, 8), dtype=torch.int64, pin_memory=True)
            lam_pin = torch.empty(ktot, dtype=torch.float64, pin_memory=True)
            st_pin.copy_(st.view(nseg, 8), non_blocking=True)
            lam_pin.copy_(lam_k, non_blocking=True)
            if hss_m:
                gam_pin = torch.empty(ktot, dtype=torch.float64, pin_memory=True)
                mu_pin = torch.empty(ktot, dtype=torch.float64, pin_memory=True)
                gam_pin.copy_(gam, non_blocking=True)
                mu_pin.copy_(mu, non_blocking=True)
            roots_ready = torch.cuda.Event()
            roots_ready.record()
            if len(big):
                # materialised-panel updates straight through the C ABI (one generator struct
                # and one shared workspace; cauchy.py's right_multiply_into per merge costs
                # ~70 us of host time each at config 5)
                kmax, kmin = int(ks[big].max()), int(ks[big].min())
                # the depth's updates run on up to DENSE_STREAMS side streams, each with its
                # own slice of the workspace (sized for the widest merge)
                nst = min(DENSE_STREAMS, len(big))
                mb = segs[big]
                # a slice holds a merge's two compacted row blocks (exact sizes: about half of
                # rows x k) and the panel workspace of the widest merge
                kt, kbn = np.maximum(ka_b, 1), np.maximum(kept[mb] - kb_b, 1)
                halves = int((n1[mb] * (kt + (kt & 1)) + n2[mb] * (kbn + (kbn & 1))).max()) + 64
                nw = nst * ((halves + int(lib.hsseig_dense_update_work_doubles(
                    kmax, max(128, DENSE_PANEL_BYTES // (8 * kmin)))) + 63) & ~31)
                pw = torch.empty(nw, **f64)
                rec9 = np.ascontiguousarray(np.stack(
                    [woff[mb], ldw[mb], nv[mb], n1[mb], koff[big], kept[mb], ka_b, kb_b, qoff[mb]], 1),
                    dtype=np.int64)
                nat.check(lib.hsseig_wave_dense_halves(
                    len(big), _cptr(rec9), nat.ptr(W), nat.ptr(dk), nat.ptr(dn), nat.ptr(gam),
                    nat.ptr(mu), nat.ptr(zh), nat.ptr(vv), nat.ptr(kperm_d), nat.ptr(Qk),
                    nat.ptr(pw), nw, nst, s), "wave_dense_halves")
            if len(tk):
                nat.check(lib.hsseig_wave_dense_update(
                    nat.ptr(W), nat.ptr(t_woff), nat.ptr(t_nv), nat.ptr(t_ldw), nat.ptr(dk),
                    nat.ptr(dn), nat.ptr(gam), nat.ptr(mu), nat.ptr(zh), nat.ptr(vv), nat.ptr(koff_d),
                    nat.ptr(Qk), nat.ptr(t_qoff), nat.ptr(t_tk), len(tk), s),
                    "wave_dense_update")
            _mark("updates_queued", depth)
            roots_ready.synchronize()
            _mark("roots_ready", depth)
            stv = st_pin.numpy()
            bad_b = (stv[:, 1] < ks) | ((ks >= 2) & (stv[:, 2] < ks))
            bad_r = stv[:, 3] < ks
            if (bad_b | bad_r).any():
                q = int(np.flatnonzero(bad_b | bad_r)[0])
                if bad_b[q]:
                    bad = int(stv[q, 1] if stv[q, 1] < ks[q] else stv[q, 2])
                    raise SecularConvergenceError(f"root {bad} lost its bracket")
                raise WeightRecomputationError(f"non-positive radicand at index {int(stv[q, 3])}")
            seg_iters = stv[:, 0]
            if hss_m:
                # the level's HSS merges, phase-batched (partition / rank from host roots)
                gam_h, mu_h, dk_h = gam_pin.numpy(), mu_pin.numpy(), d_out[kidx]
                jobs = []
                for q in sorted(hss_m):
                    m = segs[q]
                    n, k = int(nv[m]), int(kept[m])
                    sl = slice(int(koff[q]), int(koff[q + 1]))
                    C = CauchyEvecMatrix(dk[sl], gam[sl], mu[sl], zh[sl], vv[sl], dnext=dn[sl])
                    mid = int(mid_a[ms[m]])
                    rec_ = records.setdefault(mid, MergeRecord(size=n, kept=k, n_deflated=n - k))
                    Wm = W[int(woff[m]):int(woff[m + 1])].view(n, int(ldw[m]))
                    jobs.append(HssJob(Q=Wm[:, :k], C=C, seed=[cfg.seed, mid], flops=FlopCounter(),
                                       record=rec_, d=dk_h[sl], gamma=gam_h[sl], mu=mu_h[sl],
                                       out=Qk[int(qoff[m]):int(qoff[m + 1])].view(n, k),
                                       halves=(int(n1[m]),) + hss_halves[q] if q in hss_halves else None))
                update_vectors_hss_many(jobs, cfg)
                for j in jobs:
                    j.record.flops = j.flops.as_dict()
                del jobs
            lam_h = lam_pin.numpy()
        else:
            lam_h = np.zeros(0)
        # final column order of every merge
        order = np.empty(nrows, dtype=np.int64)
        lam_out = np.empty(nrows)
        koff_all = np.zeros(nm, dtype=np.int64)
        koff_all[segs] = koff[:-1]
        lib.hsseig_wave_order(nm, _cptr(roff), _cptr(kept), _cptr(koff_all), _cptr(lam_h),
                              _cptr(d_out), _cptr(order), _cptr(lam_out))
        A = torch.empty(int(ooff[-1]), **f64)
        # column descriptors: (0, Qk column) | (1, compact W column) | (2, child column)
        desc = np.empty(nrows, dtype=np.int64)
        lib.hsseig_wave_desc(nm, _cptr(roff), _cptr(kept), _cptr(order), _cptr(cmap), _cptr(src),
                             _cptr(desc))
        sel = np.flatnonzero(has_parent[ms])
        sel_left = is_left[ms[sel]]
        sel_off = np.concatenate([[0], np.cumsum(nv[sel])]).astype(np.int64)
        (g_qoff, g_kept, g_desc, ooff_d, sel_m, sel_r, sel_o) = (
            _Pack().add(qoff).add(kept).add(desc).add(ooff).add(sel, np.int32)
            .add(np.where(sel_left, nv[sel] - 1, 0)).add(sel_off[:-1]).send())
        if len(sel):
            # the rows the next depth's z needs (a left child's last row, a right child's
            # first), gathered ahead of the full gather and sent to the host behind it
            rows_d = torch.empty(int(sel_off[-1]), **f64)
            nat.check(lib.hsseig_wave_gather_rows(nat.ptr(Qk), nat.ptr(g_qoff), nat.ptr(g_kept),
                                                  nat.ptr(W), nat.ptr(woff_d), nat.ptr(wd_d),
                                                  nat.ptr(g_desc), nat.ptr(q1), nat.ptr(q2),
                                                  nat.ptr(n1_d), nat.ptr(n2_d), nat.ptr(roff_d),
                                                  nat.ptr(sel_m), nat.ptr(sel_r), nat.ptr(sel_o),
                                                  len(sel), nat.ptr(rows_d), s), "wave_gather_rows")
            rows_pin = torch.empty(int(sel_off[-1]), dtype=torch.float64, pin_memory=True)
            rows_pin.copy_(rows_d, non_blocking=True)
            ev_rows = torch.cuda.Event()
            ev_rows.record()
            pending = (ev_rows, rows_pin)
            gsel = ms[sel]
            base = len(rows_h) + sel_off[:-1]
            last_off[gsel[sel_left]] = base[sel_left]
            first_off[gsel[~sel_left]] = base[~sel_left]
        if prof is not None:
            ev_g = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev_g[0].record()
        nat.check(lib.hsseig_wave_gather(nat.ptr(Qk), nat.ptr(g_qoff), nat.ptr(g_kept),
                                         nat.ptr(W), nat.ptr(woff_d), nat.ptr(wd_d), nat.ptr(g_desc),
                                         nat.ptr(q1), nat.ptr(q2), nat.ptr(n1_d), nat.ptr(n2_d),
                                         nat.ptr(roff_d), nat.ptr(row_merge), nat.ptr(A),
                                         nat.ptr(ooff_d), nrows, s), "wave_gather")
        if prof is not None:
            ev_g[1].record()
            # bytes: every output entry written; a row reads its kept columns (dense update)
            # and its own child's share of the deflated ones (the other child's are zeros)
            prof.append(("gather", ev_g[0], ev_g[1],
                         8 * int((nv * nv + nv * kept + nv * (nv - kept) // 2).sum())))
        _mark("gather_queued", depth)
        del W, Qk
        live.pop(depth + 1, None)      # the children's blocks are dead once gathered
        live[depth] = A
        lam_all[rows] = lam_out
        qptr[ms] = np.uint64(A.data_ptr()) + (8 * ooff[:-1]).astype(np.uint64)
        # records and flop counts are built after the last depth is queued (the host is
        # otherwise the bottleneck of the deep, small-merge depths)
        pending_records.append((ms, segs, nv, kept, rho_eff, seg_iters, hss_m))
    # records and flop counts (reference conventions, dc.py:236-247)
    for ms, segs, nv, kept, rho_eff, seg_iters, hss_m in pending_records:
        for q, m in enumerate(segs.tolist()):
            mid = int(mid_a[ms[m]])
            n, k = int(nv[m]), int(kept[m])
            sec = secular_flops(k, int(seg_iters[q])) + 14 * k * k
            if q in hss_m:
                rec_ = records[mid]
                rec_.flops["secular"] = rec_.flops.get("secular", 0) + sec
            else:
                rec_ = records.setdefault(mid, MergeRecord(size=n, kept=k, n_deflated=n - k))
                rec_.flops = {"secular": sec, "update_dense": cauchy_eval_flops(k * k) + gemm_flops(n, k, k),
                              "hss_construct": 0, "hss_mult": 0}
        for m in np.flatnonzero((kept == 0) & (rho_eff != 0.0)).tolist():
            n = int(nv[m])
            records.setdefault(int(mid_a[ms[m]]), MergeRecord(size=n, kept=0, n_deflated=n)).flops = \
                {p: 0 for p in FlopCounter.PHASES}
    n = int(hi_a[-1] - lo_a[-1])
    if leaf_a[-1]:
        Q = Qbase[int(lqoff[0]):int(lqoff[0]) + n * n].view(n, n)
    else:
        Q = live[top].view(n, n)
    return lam_all, Q, records
