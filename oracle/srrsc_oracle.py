"""TEST INFRASTRUCTURE ONLY — CPU oracle for ADC1 (SRRSC HSS construction).

PARITY UNPINNED.  BASELINE.json names ADC1 ("SRRSC HSS") but the reference package
has no implementation of it (only ``dense-dc`` and ``adc-rand`` exist,
``pkg/src/hsseig/dc.py:23``), and the SRRSC papers the paper cites
 are not in the container.  This module is therefore the
*definition* the GPU path is checked against, restated from the published idea
(Gaussian elimination with complete pivoting on the generators of a Cauchy-like
matrix, whose Schur complements stay Cauchy-like), and it is validated only by
properties: the generator recurrence reproduces the explicit Schur complement,
the HSS reconstruction matches the dense Cauchy matrix to the tolerance, and full
ADC1 eigendecompositions match dense DC / closed forms.

Definition (what ``srrsc_construct`` computes).  For node t with candidate rows
R (leaf: its own indices; inner: the children's skeletons, left then right) the
block row M = C[R, t^c] (side "row") or the block column C[t^c, R]^T (side "col")
is a Cauchy-like matrix M_ab = s_a t_b / g_ab with g the stable gaps of
``hss_oracle.gaps`` (secular.py:183-203).  Step s picks the first maximum of
|M^(s)| in row-major order (complete pivoting), stops when
max|M^(s)| <= tol * max|M^(0)| or s == cap, and otherwise eliminates the pivot
(p, q) on the generators:
  side row (rows = poles i, columns = eigen indices j):
      s_i <- s_i (d_i - d_p) / g(i, q),     t_j <- t_j (lam_q - lam_j) / g(p, j)
  side col (rows = eigen indices j, columns = poles i):
      s_j <- s_j (lam_p - lam_j) / g(q, j), t_i <- t_i (d_i - d_q) / g(i, p)
with lam_a - lam_b formed through an interlacing pole (no cancellation,
``lamdiff``).  The multipliers L[a, s] = M^(s)[a, q] / M^(s)[p, q] give the
interpolation matrix X = L[:, :r] L[J, :r]^{-1} (identity on the skeleton J, in
pivot order), so M ~= X M[J, :] with error max|M^(r)|.  U / V / B / D / skeleton
indices then have exactly the meaning of the randomized tree (hss.py:151-185),
so ``hss_oracle.hss_apply_right`` multiplies either tree.
"""
from __future__ import annotations

import numpy as np

from .hss_oracle import (FLAG_TOL, Tree, f_cauchy, gaps, hss_apply_right, leaf_ranges,
                         postorder_nodes, update_dense)

MAX_WIDTH = 112     # widest tree the device slots hold (paper_1510_04591_b200/hss.py)


def _nxt(G):
    top = G.d[-1] + G.gam[-1] + G.mu[-1]
    return np.append(G.d[1:], top)


def lamdiff(G, a, b):
    """lam_a - lam_b for eigen indices a != b, through the pole between them.

    a < b: lam_a - lam_b = g(a+1, b) - mu_a,  g(a+1, b) = (d_{a+1} - d_b) - gam_b
    a > b: lam_a - lam_b = mu_b - g(b+1, a),  g(b+1, a) = (d_{b+1} - d_a) - gam_a
    Both terms carry the sign of the result.  a == b gives 0.
    """
    a = np.asarray(a, dtype=np.intp)
    b = np.asarray(b, dtype=np.intp)
    a, b = np.broadcast_arrays(a, b)
    d, gam, mu = G.d, G.gam, G.mu
    nx = _nxt(G)
    out = np.zeros(a.shape)
    lt = a < b
    gt = a > b
    out[lt] = ((nx[a[lt]] - d[b[lt]]) - gam[b[lt]]) - mu[a[lt]]
    out[gt] = mu[b[gt]] - ((nx[b[gt]] - d[a[gt]]) - gam[a[gt]])
    return out


def srrsc_block(G, cand, lo, hi, side, tol, cap, flops=None):
    """Rank-revealing Schur complement of one block row / column on its generators.

    Returns (X, J, resid, saturated, steps) with M ~= X @ M[J, :] (X identity on J).
    """
    k = G.k
    cand = np.asarray(cand, dtype=np.intp)
    comp = np.concatenate([np.arange(0, lo), np.arange(hi, k)]).astype(np.intp)
    p, n = cand.size, comp.size
    if side == "row":
        s = G.zh[cand].copy()
        t = G.v[comp].copy()
        g = gaps(cand, comp, G.d, G.gam, G.mu)
    else:
        s = G.v[cand].copy()
        t = G.zh[comp].copy()
        g = gaps(comp, cand, G.d, G.gam, G.mu).T.copy()
    L = np.zeros((p, max(cap, 1)))
    active = np.ones(p, dtype=bool)
    piv_r, piv_c = [], []
    max0 = 0.0
    r = 0
    mx = 0.0
    for step in range(cap + 1):
        M = (s[:, None] * t[None, :]) / g if p and n else np.zeros((p, n))
        A = np.abs(M)
        if flops is not None:
            flops.hss_construct += f_cauchy(A.size)
        if A.size:
            flat = int(np.argmax(A))
            mx = float(A.flat[flat])
        else:
            flat, mx = 0, 0.0
        if step == 0:
            max0 = mx
        if mx == 0.0 or mx <= tol * max0 or step == cap:
            r = step
            break
        a, b = divmod(flat, n)
        pv = M[a, b]
        col = M[:, b] / pv
        col[~active] = 0.0
        col[a] = 1.0
        L[:, step] = col
        # generator updates (row factors use column b of the gaps, column factors row a)
        if side == "row":
            rf = (G.d[cand] - G.d[cand[a]]) / g[:, b]
            cf = lamdiff(G, comp[b], comp) / g[a, :]
        else:
            rf = lamdiff(G, cand[a], cand) / g[:, b]
            cf = (G.d[comp] - G.d[comp[b]]) / g[a, :]
        s = s * rf
        t = t * cf
        s[a] = 0.0
        t[b] = 0.0
        active[a] = False
        piv_r.append(a)
        piv_c.append(b)
    J = np.asarray(piv_r, dtype=np.intp)
    X = np.zeros((p, r))
    if r:
        L11 = L[J, :r]
        Xr = L[:, :r].copy()
        for tt in range(r - 1, -1, -1):        # x L11 = l, L11 unit lower triangular
            if tt + 1 < r:
                Xr[:, tt] -= Xr[:, tt + 1:r] @ L11[tt + 1:r, tt]
        X[:] = Xr
        X[J, :] = 0.0
        X[J, np.arange(r)] = 1.0
        if flops is not None:
            flops.hss_construct += p * r * r
    resid = mx / max0 if max0 > 0.0 else 0.0
    sat = bool(r == cap and cap > 0 and resid > FLAG_TOL)
    return X, J, resid, sat, r


def srrsc_construct(G, ranges, cap, tol, flops=None):
    """ADC1: HSS tree of the Cauchy-like eigenvector matrix from its generators alone."""
    if len(ranges) < 2:
        raise ValueError("need at least two leaves")
    if cap < 1:
        raise ValueError("need a rank cap >= 1")
    nodes, root = postorder_nodes(ranges)
    tree = Tree(nodes, root, list(ranges), G.k)
    for lev in range(max(n.level for n in nodes), 0, -1):
        for nd in (n for n in nodes if n.level == lev):
            if nd.leaf:
                t = np.arange(nd.lo, nd.hi)
                nd.D = G.block(t, t, flops)
                rc, cc = t, t
            else:
                a, b = nodes[nd.left], nodes[nd.right]
                a.B = G.block(a.rsel, b.csel, flops)
                b.B = G.block(b.rsel, a.csel, flops)
                rc = np.concatenate([a.rsel, b.rsel])
                cc = np.concatenate([a.csel, b.csel])
            for side, cand in (("row", rc), ("col", cc)):
                X, J, res, sat, _ = srrsc_block(G, cand, nd.lo, nd.hi, side, tol, cap, flops)
                if sat:
                    tree.flagged = True
                    tree.flags.append((nd.idx, side, float(res)))
                if side == "row":
                    nd.U, nd.rloc, nd.rres, nd.rsel = X, J, res, cand[J]
                else:
                    nd.V, nd.cloc, nd.cres, nd.csel = X, J, res, cand[J]
    top = nodes[root]
    a, b = nodes[top.left], nodes[top.right]
    a.B = G.block(a.rsel, b.csel, flops)
    b.B = G.block(b.rsel, a.csel, flops)
    ranks = [n.U.shape[1] for n in nodes if n.U is not None] + \
            [n.V.shape[1] for n in nodes if n.V is not None]
    tree.r_used = max(ranks) if ranks else 0
    return tree


def srrsc_cap(ranges):
    """Rank cap of ADC1: the smallest leaf (bounded by the device slot width)."""
    return min(min(hi - lo for lo, hi in ranges), MAX_WIDTH)


def update_srrsc(Qb, G, leaf, tol, flops=None, info=None, return_tree=False):
    """ADC1 merge update: partition (hss.py:48-79), SRRSC tree, flag -> dense fallback, multiply."""
    def fallback():
        if info is not None:
            info.used_hss, info.fell_back = False, True
        out = update_dense(Qb, G, flops)
        return (out, None) if return_tree else out

    try:
        ranges = leaf_ranges(G.k, leaf, G.mu)
    except ValueError:
        return fallback()
    T = srrsc_construct(G, ranges, srrsc_cap(ranges), tol, flops)
    if T.flagged:
        return fallback()
    if info is not None:
        info.used_hss, info.hss_rank = True, T.r_used
    out = hss_apply_right(Qb, T, flops)
    return (out, T) if return_tree else out
