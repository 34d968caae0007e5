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
from .cauchy import DENSE_PANEL_MIN_K, CauchyEvecMatrix
from .dc import (BaseCaseError, EigenResult, MergeRecord, SolverConfig, merge_update,
                 update_vectors_hss)
from .flops import FlopCounter, cauchy_eval_flops, gemm_flops, secular_flops
from .secular import SecularConvergenceError, WeightRecomputationError

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
    aa = np.concatenate([a_mod[lo:hi] for lo, hi in leaves])
    a_d, b_d, off_d, qoff_d = _f64(aa), _f64(bb), _i64(off), _i64(qoff)
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
def _tree(n, base):
    """Recursion nodes (dc.py:194-203): split at n // 2, merge ids in postorder."""
    nodes = []
    ids = itertools.count()

    def rec(lo, hi, depth):
        if hi - lo <= base:
            nodes.append({"lo": lo, "hi": hi, "depth": depth, "leaf": True})
            return len(nodes) - 1
        m = lo + (hi - lo) // 2
        left = rec(lo, m, depth + 1)
        right = rec(m, hi, depth + 1)
        nodes.append({"lo": lo, "hi": hi, "depth": depth, "leaf": False, "left": left,
                      "right": right, "split": m, "mid": next(ids)})
        return len(nodes) - 1

    root = rec(0, n, 0)
    return nodes, root


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
    a_mod, _ = _plan(a, b, cfg.base_size)
    nodes, root = _tree(T.n, cfg.base_size)
    lam, Q, records = solve_subtree(a_mod, b, nodes, root, cfg)
    flops = FlopCounter()
    merges = [records[k] for k in sorted(records)]
    for r in merges:
        for p_ in FlopCounter.PHASES:
            setattr(flops, p_, getattr(flops, p_) + r.flops.get(p_, 0))
    return EigenResult(lam=lam, Q=Q, merges=merges, flops=flops)


def _subtree_nodes(nodes, sub):
    out = []
    stack = [sub]
    while stack:
        i = stack.pop()
        out.append(i)
        if not nodes[i]["leaf"]:
            stack += [nodes[i]["left"], nodes[i]["right"]]
    return set(out)


def solve_subtree(a_mod, b, nodes, sub, cfg):
    """Eigenpairs of the recursion node `sub` (its base cases and every merge below it,
    level-batched); a_mod carries all split modifications (_plan).  Returns (lam host,
    Q device n x n in the node's local coordinates, {merge id: MergeRecord})."""
    lib = nat.load()
    s = nat.stream_ptr()
    f64 = dict(dtype=torch.float64, device="cuda")
    members = _subtree_nodes(nodes, sub)
    leaf_ids = sorted((i for i in members if nodes[i]["leaf"]), key=lambda i: nodes[i]["lo"])
    base = _base_cases(a_mod, b, [(nodes[i]["lo"], nodes[i]["hi"]) for i in leaf_ids], s)
    state = {}       # node -> (lam host, Q device view n x n)
    for i in leaf_ids:
        state[i] = base[(nodes[i]["lo"], nodes[i]["hi"])]
    records = {}
    bm = ctypes.c_int32(0)
    bn = ctypes.c_int32(0)
    lib.hsseig_wave_tile_shape(ctypes.byref(bm), ctypes.byref(bn))
    bm, bn = bm.value, bn.value
    maxdepth = max(nodes[i]["depth"] for i in members)
    for depth in range(maxdepth - 1, -1, -1):
        ms = [i for i in sorted(members) if nodes[i]["depth"] == depth and not nodes[i]["leaf"]]
        if not ms:
            continue
        nm = len(ms)
        n1 = np.array([nodes[i]["split"] - nodes[i]["lo"] for i in ms], dtype=np.int64)
        n2 = np.array([nodes[i]["hi"] - nodes[i]["split"] for i in ms], dtype=np.int64)
        nv = n1 + n2
        roff = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
        nrows = int(roff[-1])
        kids = [(state.pop(nodes[i]["left"]), state.pop(nodes[i]["right"])) for i in ms]
        L = np.concatenate([np.concatenate([c1[0], c2[0]]) for c1, c2 in kids])
        q1 = _u64([c1[1].data_ptr() for c1, _ in kids])
        q2 = _u64([c2[1].data_ptr() for _, c2 in kids])
        n1_d, n2_d, nv_d, roff_d = _i64(n1), _i64(n2), _i64(nv), _i64(roff)
        # boundary rows -> host (sync 1)
        zrow_d = torch.empty(nrows, **f64)
        nat.check(lib.hsseig_wave_zrows(nat.ptr(q1), nat.ptr(q2), nat.ptr(n1_d), nat.ptr(n2_d),
                                        nat.ptr(roff_d), nm, nat.ptr(zrow_d), s), "wave_zrows")
        zrow = zrow_d.cpu().numpy()
        bk = np.array([b[nodes[i]["split"] - 1] for i in ms], dtype=np.float64)
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
        W = torch.empty(max(int(woff[-1]), 2), **f64)
        woff_d, wd_d = _i64(woff), _i64(wd)
        # (device temporaries stay referenced until their launch: a freed block is reused
        #  by the next upload on the same stream)
        row_merge = _i32(np.repeat(np.arange(nm), nv))
        csrc_d, coff_d = _i64(csrc[:max(int(coff[-1]), 1)]), _i64(coff)
        nat.check(lib.hsseig_wave_assemble(nat.ptr(q1), nat.ptr(q2), nat.ptr(n1_d), nat.ptr(n2_d),
                                           nat.ptr(roff_d), nat.ptr(row_merge), nat.ptr(csrc_d),
                                           nat.ptr(coff_d), nat.ptr(wd_d), nat.ptr(W), nat.ptr(woff_d),
                                           nrows, s), "wave_assemble")
        nrot = int(rot_off[-1])
        if nrot:
            rot_d = (_i64(rot_off), _i64(ca[:nrot]), _i64(cb[:nrot]), _f64(rc[:nrot]),
                     _f64(rs[:nrot]))
            nat.check(lib.hsseig_wave_rotate(nat.ptr(W), nat.ptr(woff_d), nat.ptr(nv_d), nat.ptr(wd_d),
                                             *(nat.ptr(t) for t in rot_d), nm, int(nv.max()), s),
                      "wave_rotate")
        # the kept rank-one systems, concatenated
        segs = np.flatnonzero(kept > 0)
        nseg = len(segs)
        ks = kept[segs]
        koff = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
        kidx = np.repeat(roff[segs] - koff[:-1], ks) + np.arange(ktot)
        qoff = np.concatenate([[0], np.cumsum(nv * kept)]).astype(np.int64)
        Qk = torch.empty(max(int(qoff[-1]), 1), **f64)
        hss_m = set()
        seg_iters = np.zeros(nseg, dtype=np.int64)
        if nseg:
            dk, zk = _f64(d_out[kidx]), _f64(z_out[kidx])
            koff_d, seg_of = _i64(koff), _i32(np.repeat(np.arange(nseg), ks))
            rho_d = _f64(rho_eff[segs])
            lam_k, gam, mu, dn, zh, vv = (torch.empty(ktot, **f64) for _ in range(6))
            its = torch.empty(ktot, dtype=torch.int32, device="cuda")
            st0 = np.zeros((nseg, 8), dtype=np.int64)
            st0[:, 1:4] = ks[:, None]
            st = torch.as_tensor(st0, device="cuda")
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
            # dense updates of every system not taking the HSS path: the large ones through
            # materialised C panels on the TMA/DMMA engine, the rest grouped in one launch
            tasks = []
            big = []
            for q, m in enumerate(segs):
                n, k = int(nv[m]), int(kept[m])
                if cfg.method == "adc-rand" and k > cfg.hss_threshold:
                    hss_m.add(q)
                    continue
                if k >= DENSE_PANEL_MIN_K:
                    big.append(q)
                    continue
                mt, nt = -(-n // bm), -(-k // bn)
                t = np.empty((mt * nt, 3), dtype=np.int32)
                t[:, 0] = q
                t[:, 1] = np.repeat(np.arange(mt), nt)
                t[:, 2] = np.tile(np.arange(nt), mt)
                tasks.append(t)
            for q in big:
                m = segs[q]
                n, k = int(nv[m]), int(kept[m])
                sl = slice(int(koff[q]), int(koff[q + 1]))
                C = CauchyEvecMatrix(dk[sl], gam[sl], mu[sl], zh[sl], vv[sl], dnext=dn[sl])
                Wm = W[int(woff[m]):int(woff[m + 1])].view(n, int(ldw[m]))
                C.right_multiply_into(Wm[:, :k], out=Qk[int(qoff[m]):int(qoff[m + 1])].view(n, k))
            if tasks:
                tk = np.concatenate(tasks)
                dd_ = (_i64(woff[segs]), _i64(nv[segs]), _i64(qoff[segs]), _i32(tk.ravel()),
                       _i64(ldw[segs]))
                nat.check(lib.hsseig_wave_dense_update(
                    nat.ptr(W), nat.ptr(dd_[0]), nat.ptr(dd_[1]), nat.ptr(dd_[4]), nat.ptr(dk),
                    nat.ptr(dn), nat.ptr(gam), nat.ptr(mu), nat.ptr(zh), nat.ptr(vv), nat.ptr(koff_d),
                    nat.ptr(Qk), nat.ptr(dd_[2]), nat.ptr(dd_[3]), len(tk), s),
                    "wave_dense_update")
            # statuses + roots (sync 2)
            stv = st.cpu().numpy()
            for q, m in enumerate(segs):
                k = int(ks[q])
                if stv[q, 1] < k or (k >= 2 and stv[q, 2] < k):
                    bad = int(stv[q, 1] if stv[q, 1] < k else stv[q, 2])
                    raise SecularConvergenceError(f"root {bad} lost its bracket")
                if stv[q, 3] < k:
                    raise WeightRecomputationError(f"non-positive radicand at index {int(stv[q, 3])}")
            seg_iters = stv[:, 0]
            for q in sorted(hss_m):
                m = segs[q]
                n, k = int(nv[m]), int(kept[m])
                sl = slice(int(koff[q]), int(koff[q + 1]))
                C = CauchyEvecMatrix(dk[sl], gam[sl], mu[sl], zh[sl], vv[sl], dnext=dn[sl])
                nd = nodes[ms[m]]
                rec_ = records.setdefault(nd["mid"], MergeRecord(size=n, kept=k, n_deflated=n - k))
                fc = FlopCounter()
                Wm = W[int(woff[m]):int(woff[m + 1])].view(n, int(ldw[m]))
                out = update_vectors_hss(Wm[:, :k], C, cfg, seed=[cfg.seed, nd["mid"]], flops=fc,
                                         record=rec_)
                Qk[int(qoff[m]):int(qoff[m + 1])].view(n, k).copy_(out)
                rec_.flops = fc.as_dict()
                del out
            lam_h = lam_k.cpu().numpy()
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
        ooff_d = _i64(ooff)
        # column descriptors: (0, Qk column) | (1, compact W column) | (2, child column)
        rm = np.repeat(np.arange(nm), nv)
        pg = order + roff[rm]
        cmg = cmap[pg]
        desc = np.where(order < kept[rm], order,
                        np.where(cmg >= 0, (1 << 40) | cmg, (2 << 40) | src[pg])).astype(np.int64)
        g_ = (_i64(qoff), _i64(kept), _i64(desc))
        nat.check(lib.hsseig_wave_gather(nat.ptr(Qk), nat.ptr(g_[0]), nat.ptr(g_[1]),
                                         nat.ptr(W), nat.ptr(woff_d), nat.ptr(wd_d), nat.ptr(g_[2]),
                                         nat.ptr(q1), nat.ptr(q2), nat.ptr(n1_d), nat.ptr(n2_d),
                                         nat.ptr(roff_d), nat.ptr(row_merge), nat.ptr(A),
                                         nat.ptr(ooff_d), nrows, s), "wave_gather")
        del W, Qk, kids, q1, q2      # the children's blocks are dead once gathered
        # records and flop counts (reference conventions, dc.py:236-247)
        for q, m in enumerate(segs):
            nd = nodes[ms[m]]
            n, k = int(nv[m]), int(kept[m])
            sec = secular_flops(k, int(seg_iters[q])) + 14 * k * k
            if q in hss_m:
                rec_ = records[nd["mid"]]
                rec_.flops["secular"] = rec_.flops.get("secular", 0) + sec
            else:
                rec_ = records.setdefault(nd["mid"], MergeRecord(size=n, kept=k, n_deflated=n - k))
                rec_.flops = {"secular": sec, "update_dense": cauchy_eval_flops(k * k) + gemm_flops(n, k, k),
                              "hss_construct": 0, "hss_mult": 0}
        for m in range(nm):
            nd = nodes[ms[m]]
            n = int(nv[m])
            if kept[m] == 0 and rho_eff[m] != 0.0:
                records.setdefault(nd["mid"], MergeRecord(size=n, kept=0, n_deflated=n)).flops = \
                    {p: 0 for p in FlopCounter.PHASES}
            state[ms[m]] = (lam_out[roff[m]:roff[m + 1]].copy(),
                            A[int(ooff[m]):int(ooff[m + 1])].view(n, n))
    lam, Q = state[sub]
    return lam, Q, records
