"""TEST INFRASTRUCTURE ONLY — CPU oracle for the DC merge-step hot path.

A NumPy/SciPy restatement of the reference package ``hsseig`` (arXiv 1510.04591
reference, ``/root/reference/pkg/src/hsseig``) for every function on the
merge path.  Each function cites the reference ``file:line`` it restates.
The compiled pieces (secular roots, base-case QL) come from ``oracle_c.c``
through ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``).

Third-party arithmetic the reference delegates (restated by calling the same
libraries): LAPACK ``dgeqp3`` / ``dtrtrs`` through SciPy, BLAS ``dgemm`` through
NumPy, and NumPy's PCG64 + ziggurat ``standard_normal`` for the sample block.
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

EPS = float(np.finfo(np.float64).eps)
_HERE = os.path.dirname(os.path.abspath(__file__))

# constants of pkg/src/hsseig/hss.py:20-24
SHIFT_GAP = 1e-10
SHIFT_REACH = 5
RANK_CAP = 100
ID_TOL = 1e-15
FLAG_TOL = 1e-12
DENSE_LIMIT = 4096


class SecularConvergenceError(ArithmeticError):
    """pkg/src/hsseig/secular.py:25"""


class WeightRecomputationError(ArithmeticError):
    """pkg/src/hsseig/secular.py:29"""


class BaseCaseError(ArithmeticError):
    """pkg/src/hsseig/dc.py:27"""


# ---------------------------------------------------------------------------
# compiled oracle pieces
# ---------------------------------------------------------------------------
_lib = None


def _clib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        P = ctypes.POINTER(ctypes.c_double)
        lib.oracle_secular_all.restype = ctypes.c_int64
        lib.oracle_secular_all.argtypes = [P, P, ctypes.c_int64, ctypes.c_double, P, P, P,
                                           ctypes.POINTER(ctypes.c_int64)]
        lib.oracle_tql2.restype = ctypes.c_int
        lib.oracle_tql2.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int]
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def secular_all(d, z, rho, per_root=False):
    """Roots + gap pairs; restates pkg/src/hsseig/_kernels.pyx:178-234."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    k = d.size
    lam, gam, mu = np.empty(k), np.empty(k), np.empty(k)
    its = np.zeros(k, dtype=np.int64)
    total = _clib().oracle_secular_all(_dp(d), _dp(z), k, float(rho), _dp(lam), _dp(gam),
                                       _dp(mu), its.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if per_root:
        return lam, gam, mu, int(total), its
    return lam, gam, mu, int(total)


def tql2(d, e, Z, max_iter=30):
    """In-place implicit QL; restates pkg/src/hsseig/_kernels.pyx:352-411."""
    assert d.flags.c_contiguous and Z.flags.c_contiguous
    e = np.ascontiguousarray(e, dtype=np.float64)
    if e.size == 0:
        e = np.zeros(1)
    return _clib().oracle_tql2(_dp(d), _dp(e), _dp(Z), d.size, int(max_iter))


# ---------------------------------------------------------------------------
# flop conventions (pkg/src/hsseig/flops.py:14-49)
# ---------------------------------------------------------------------------
@dataclass
class Flops:
    secular: int = 0
    update_dense: int = 0
    hss_construct: int = 0
    hss_mult: int = 0

    def as_dict(self):
        return dict(secular=self.secular, update_dense=self.update_dense,
                    hss_construct=self.hss_construct, hss_mult=self.hss_mult)


def f_gemm(m, n, p):
    return 2 * m * n * p


def f_cauchy(entries):
    return 6 * entries


def f_cpqr(m, n, r):
    return 4 * m * n * r


# ---------------------------------------------------------------------------
# secular stage (pkg/src/hsseig/secular.py)
# ---------------------------------------------------------------------------
def solve_roots(d, z, rho, flops=None):
    """secular.py:159-180 — roots, then the bracket-loss check on gamma/mu."""
    k = len(d)
    if k == 0:
        raise ValueError("empty system")
    lam, gam, mu, iters = secular_all(d, z, rho)
    if flops is not None:
        flops.secular += 10 * k * iters
    bad = np.flatnonzero(gam <= 0.0)
    if bad.size == 0 and k >= 2:
        bad = np.flatnonzero(mu <= 0.0)
    if bad.size:
        raise SecularConvergenceError(f"root {int(bad[0])} lost its bracket")
    return lam, gam, mu, iters


def gaps(rows, cols, d, gam, mu):
    """d[i] - lam[j] via the i<=j / i>j branches (secular.py:183-203)."""
    rows = np.asarray(rows, dtype=np.intp)
    cols = np.asarray(cols, dtype=np.intp)
    top = d[-1] + gam[-1] + mu[-1]          # virtual pole closing the last interval
    nxt = np.append(d[1:], top)             # d[j+1], with the virtual pole at j=k-1
    di = d[rows][:, None]
    left = (di - d[cols][None, :]) - gam[cols][None, :]
    right = (di - nxt[cols][None, :]) + mu[cols][None, :]
    return np.where(rows[:, None] <= cols[None, :], left, right)


def loewner(d, gam, mu, z, rho, flops=None, block=512):
    """Recomputed weights (secular.py:206-236)."""
    k = d.size
    zh = np.empty(k)
    allc = np.arange(k)
    for s in range(0, k, block):
        rr = np.arange(s, min(s + block, k))
        numer = -gaps(rr, allc, d, gam, mu)
        denom = d[None, :] - d[rr][:, None]
        q = np.ones_like(numer)
        np.divide(numer, denom, out=q, where=denom != 0.0)
        q[rr - s, rr] = 1.0
        rad = np.prod(q, axis=1) * gam[rr] / rho
        badm = (rad <= 0.0) | ~np.isfinite(rad)
        if badm.any():
            raise WeightRecomputationError(
                f"non-positive radicand at index {int(rr[np.flatnonzero(badm)[0]])}")
        zh[rr] = np.sqrt(rad)
    if flops is not None:
        flops.secular += 8 * k * k
    return np.copysign(zh, z)


def normalizers(d, gam, mu, zh, flops=None, block=512):
    """v_j = 1/||zhat / (d - lam_j)|| (secular.py:239-250)."""
    k = d.size
    v = np.empty(k)
    allr = np.arange(k)
    for s in range(0, k, block):
        cc = np.arange(s, min(s + block, k))
        g = gaps(allr, cc, d, gam, mu)
        v[cc] = 1.0 / np.sqrt(((zh[:, None] / g) ** 2).sum(axis=0))
    if flops is not None:
        flops.secular += 6 * k * k
    return v


@dataclass
class Generators:
    """Cauchy-like eigenvector matrix held by generators (cauchy.py:15-38)."""
    d: np.ndarray
    gam: np.ndarray
    mu: np.ndarray
    zh: np.ndarray
    v: np.ndarray

    @property
    def k(self):
        return self.d.size

    def block(self, rows, cols, flops=None, phase="hss_construct"):
        """cauchy.py:48-56"""
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        out = (self.zh[rows][:, None] * self.v[cols][None, :]) / gaps(rows, cols, self.d, self.gam, self.mu)
        if flops is not None:
            setattr(flops, phase, getattr(flops, phase) + f_cauchy(out.size))
        return out

    def dense(self, flops=None, phase="hss_construct"):
        idx = np.arange(self.k)
        return self.block(idx, idx, flops, phase)

    def times(self, X, flops=None, block=512):
        """C @ X (cauchy.py:70-84)."""
        k = self.k
        out = np.empty((k, X.shape[1]))
        allc = np.arange(k)
        for s in range(0, k, block):
            rr = np.arange(s, min(s + block, k))
            out[rr] = self.block(rr, allc) @ X
        if flops is not None:
            flops.hss_construct += f_gemm(k, k, X.shape[1]) + f_cauchy(k * k)
        return out

    def t_times(self, X, flops=None, block=512):
        """C^T @ X (cauchy.py:86-100)."""
        k = self.k
        out = np.zeros((k, X.shape[1]))
        allc = np.arange(k)
        for s in range(0, k, block):
            rr = np.arange(s, min(s + block, k))
            out += self.block(rr, allc).T @ X[rr]
        if flops is not None:
            flops.hss_construct += f_gemm(k, k, X.shape[1]) + f_cauchy(k * k)
        return out


def generators_from_roots(d, z, rho, flops=None):
    """solve_secular -> recompute_weights -> from_secular (dc.py:238-240)."""
    lam, gam, mu, iters = solve_roots(d, z, rho, flops)
    zh = loewner(d, gam, mu, z, rho, flops)
    v = normalizers(d, gam, mu, zh, flops)
    return Generators(np.asarray(d, dtype=np.float64), gam, mu, zh, v), lam, iters


# ---------------------------------------------------------------------------
# HSS partition and rank estimate (hss.py:48-103)
# ---------------------------------------------------------------------------
def leaf_ranges(k, m, mu=None):
    """Power-of-two leaf count, near-equal sizes, clustered boundaries nudged (hss.py:48-79)."""
    if k < 2 * m:
        raise ValueError(f"order {k} below twice the leaf size {m}")
    nl = 1
    while nl * m < k:
        nl *= 2
    q, extra = divmod(k, nl)
    bounds = np.zeros(nl + 1, dtype=np.int64)
    bounds[1:] = np.cumsum([q + 1] * extra + [q] * (nl - extra))
    if mu is not None and nl > 1:
        for b in range(1, nl):
            s = int(bounds[b])
            if mu[s - 1] >= SHIFT_GAP:
                continue
            cand = np.arange(max(bounds[b - 1] + 1, s - SHIFT_REACH),
                             min(bounds[b + 1] - 1, s + SHIFT_REACH) + 1)
            gapsb = mu[cand - 1]
            if float(gapsb.max()) > mu[s - 1]:
                bounds[b] = cand[int(np.argmax(gapsb))]
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(nl)]


def exp_sum_terms(R, eps):
    """hss.py:82-84"""
    return int(math.ceil(math.log(16.0 / eps) * math.log(8.0 * R) / math.pi ** 2))


def rank_estimate(ranges, d, gam, mu, eps=1e-16, cap=RANK_CAP):
    """hss.py:87-103"""
    if len(ranges) < 2:
        return 0
    span = (d[-1] + gam[-1]) - d[0]
    best = 0
    for lo, _ in ranges[1:]:
        best = max(best, exp_sum_terms(max(span / mu[lo - 1], 1.0), eps))
    return min(max(best, 1), cap)


# ---------------------------------------------------------------------------
# interpolative decomposition (hss.py:106-148)
# ---------------------------------------------------------------------------
def row_id(M, tol, max_rank):
    """M ~= X @ M[J]; returns (X, J, resid, saturated) per hss.py:120-148."""
    p, w = M.shape
    nf = float(np.linalg.norm(M, "fro"))
    if nf == 0.0 or p == 0 or w == 0 or max_rank == 0:
        return np.zeros((p, 0)), np.zeros(0, dtype=np.intp), 0.0, False
    _, R, piv = scipy.linalg.qr(M.T, mode="economic", pivoting=True)
    mass = np.append(np.cumsum((R * R).sum(axis=1)[::-1])[::-1], 0.0)
    cut = (tol * nf) ** 2
    want = int(np.searchsorted(-mass, -cut))
    nz = int(np.count_nonzero(np.abs(np.diag(R)) > 0.0))
    r = min(want, max_rank, nz)
    sat = bool(want >= max_rank and math.sqrt(max(mass[max_rank - 1], 0.0)) > FLAG_TOL * nf)
    resid = math.sqrt(max(mass[r], 0.0)) / nf
    coef = scipy.linalg.solve_triangular(R[:r, :r], R[:r, r:])
    X = np.zeros((p, r))
    X[piv[:r], np.arange(r)] = 1.0
    X[piv[r:], :] = coef.T
    return X, piv[:r].astype(np.intp), resid, sat


# ---------------------------------------------------------------------------
# HSS tree, randomized construction and the structured product
# ---------------------------------------------------------------------------
@dataclass
class Node:
    idx: int
    level: int
    lo: int
    hi: int
    left: int = -1
    right: int = -1
    parent: int = -1
    sibling: int = -1
    D: np.ndarray | None = None
    U: np.ndarray | None = None
    V: np.ndarray | None = None
    B: np.ndarray | None = None
    rsel: np.ndarray | None = None      # global skeleton rows
    csel: np.ndarray | None = None      # global skeleton columns
    rloc: np.ndarray | None = None
    cloc: np.ndarray | None = None
    rres: float = 0.0
    cres: float = 0.0

    @property
    def leaf(self):
        return self.left < 0


@dataclass
class Tree:
    nodes: list
    root: int
    ranges: list
    k: int
    r_used: int = 0
    flagged: bool = False
    flags: list = field(default_factory=list)

    def by_level(self):
        depth = max(n.level for n in self.nodes)
        out = [[] for _ in range(depth + 1)]
        for n in self.nodes:
            out[n.level].append(n.idx)
        return out


def postorder_nodes(ranges):
    """Postorder full binary tree over the leaf ranges (hss.py:188-214)."""
    nodes = []

    def grow(a, b, lev):
        if b - a == 1:
            nodes.append(Node(len(nodes), lev, *ranges[a]))
            return len(nodes) - 1
        h = (a + b) // 2
        L = grow(a, h, lev + 1)
        R = grow(h, b, lev + 1)
        nodes.append(Node(len(nodes), lev, nodes[L].lo, nodes[R].hi, left=L, right=R))
        me = len(nodes) - 1
        nodes[L].parent = nodes[R].parent = me
        nodes[L].sibling, nodes[R].sibling = R, L
        return me

    root = grow(0, len(ranges), 0)
    return nodes, root


def sample_block(k, w, seed):
    """The Gaussian sample the reference draws (hss.py:236-237)."""
    return np.random.default_rng(seed).standard_normal((k, w))


# The B200 path's sample (DESIGN.md §2 "off-diagonal sample"): Phi_t = C(t, t^c) Omega(t^c)
# formed directly instead of Y_t - D_t Omega_t, which cancels the dominant diagonal block and
# leaves the sample's rounding noise for the ID to truncate against.  Not the reference's
# arithmetic; rand_construct(offdiag=True) defines what the GPU's default mode computes.
def offdiag_samples(G, ranges, X):
    """(Phi, Theta) with Phi[t] = C(t, t^c) X(t^c), Theta[t] = C(t^c, t)^T X(t^c) per leaf t."""
    k = G.k
    allc = np.arange(k)
    Phi = np.empty((k, X.shape[1]))
    The = np.empty((k, X.shape[1]))
    for lo, hi in ranges:
        t = np.arange(lo, hi)
        off = np.concatenate([allc[:lo], allc[hi:]])
        Phi[lo:hi] = G.block(t, off) @ X[off]
        The[lo:hi] = G.block(off, t).T @ X[off]
    return Phi, The


def rand_construct(G, ranges, r, p=10, seed=0, id_tol=ID_TOL, flops=None, Omega=None,
                   offdiag=False):
    """Algorithm 2 with one sample block for both sides (hss.py:217-306); offdiag=True
    forms the leaf samples without the diagonal-block cancellation (offdiag_samples)."""
    if len(ranges) < 2:
        raise ValueError("need at least two leaves")
    if r < 1 or p < 0:
        raise ValueError("need rank estimate >= 1 and oversampling >= 0")
    w = r + p
    if w > min(hi - lo for lo, hi in ranges):
        raise ValueError("sample width exceeds smallest leaf")
    if Omega is None:
        Omega = sample_block(G.k, w, seed)
    if offdiag:
        Y, Z = offdiag_samples(G, ranges, Omega)
        if flops is not None:
            flops.hss_construct += 2 * (f_gemm(G.k, G.k, Omega.shape[1]) + f_cauchy(G.k * G.k))
    else:
        Y = G.times(Omega, flops)
        Z = G.t_times(Omega, flops)
    nodes, root = postorder_nodes(ranges)
    tree = Tree(nodes, root, list(ranges), G.k)
    psel, tsel, ycomp, zcomp = {}, {}, {}, {}

    def do_id(M, side, nd):
        X, J, res, sat = row_id(M, id_tol, w)
        if flops is not None:
            flops.hss_construct += f_cpqr(M.shape[1], M.shape[0], max(X.shape[1], 1))
        if sat:
            tree.flagged = True
            tree.flags.append((nd.idx, side, float(res)))
        return X, J, res

    for lev in range(max(n.level for n in nodes), 0, -1):
        for nd in (n for n in nodes if n.level == lev):
            if nd.leaf:
                t = np.arange(nd.lo, nd.hi)
                nd.D = G.block(t, t, flops)
                Om = Omega[nd.lo:nd.hi]
                if offdiag:
                    Phi, The = Y[nd.lo:nd.hi], Z[nd.lo:nd.hi]
                else:
                    Phi = Y[nd.lo:nd.hi] - nd.D @ Om
                    The = Z[nd.lo:nd.hi] - nd.D.T @ Om
                if flops is not None:
                    flops.hss_construct += 2 * f_gemm(t.size, t.size, w)
                nd.U, nd.rloc, nd.rres = do_id(Phi, "row", nd)
                nd.V, nd.cloc, nd.cres = do_id(The, "col", nd)
                nd.rsel, nd.csel = nd.lo + nd.rloc, nd.lo + nd.cloc
                ycomp[nd.idx] = nd.V.T @ Om
                zcomp[nd.idx] = nd.U.T @ Om
            else:
                a, b = nodes[nd.left], nodes[nd.right]
                a.B = G.block(a.rsel, b.csel, flops)
                b.B = G.block(b.rsel, a.csel, flops)
                Phi = np.vstack([psel[a.idx] - a.B @ ycomp[b.idx], psel[b.idx] - b.B @ ycomp[a.idx]])
                The = np.vstack([tsel[a.idx] - b.B.T @ zcomp[b.idx], tsel[b.idx] - a.B.T @ zcomp[a.idx]])
                if flops is not None:
                    flops.hss_construct += 2 * f_gemm(Phi.shape[0], w, max(a.B.shape))
                nd.U, nd.rloc, nd.rres = do_id(Phi, "row", nd)
                nd.V, nd.cloc, nd.cres = do_id(The, "col", nd)
                nd.rsel = np.concatenate([a.rsel, b.rsel])[nd.rloc]
                nd.csel = np.concatenate([a.csel, b.csel])[nd.cloc]
                ycomp[nd.idx] = nd.V.T @ np.vstack([ycomp[a.idx], ycomp[b.idx]])
                zcomp[nd.idx] = nd.U.T @ np.vstack([zcomp[a.idx], zcomp[b.idx]])
            psel[nd.idx] = Phi[nd.rloc]
            tsel[nd.idx] = The[nd.cloc]
    top = nodes[root]
    a, b = nodes[top.left], nodes[top.right]
    a.B = G.block(a.rsel, b.csel, flops)
    b.B = G.block(b.rsel, a.csel, flops)
    ranks = [n.U.shape[1] for n in nodes if n.U is not None] + \
            [n.V.shape[1] for n in nodes if n.V is not None]
    tree.r_used = max(ranks) if ranks else 0
    return tree


def hss_apply_right(X, T, flops=None):
    """X @ H by upsweep / downsweep / leaf finish (hss.py:309-361, PAPER Alg. 3)."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if X.shape[1] != T.k:
        raise ValueError("width mismatch")
    P = X.shape[0]
    nodes = T.nodes
    lv = T.by_level()
    G = {}
    for lev in range(len(lv) - 1, 0, -1):
        for i in lv[lev]:
            nd = nodes[i]
            A = X[:, nd.lo:nd.hi] if nd.leaf else np.hstack([G[nd.left], G[nd.right]])
            G[i] = A @ nd.U
            if flops is not None:
                flops.hss_mult += f_gemm(P, A.shape[1], nd.U.shape[1])
    out = np.empty_like(X)
    carry = {}
    for lev in range(1, len(lv)):
        for i in lv[lev]:
            nd = nodes[i]
            sb = nodes[nd.sibling]
            F = G[nd.sibling] @ sb.B
            if flops is not None:
                flops.hss_mult += f_gemm(P, *sb.B.shape)
            if i in carry:
                F = F + carry.pop(i)
            if nd.leaf:
                out[:, nd.lo:nd.hi] = X[:, nd.lo:nd.hi] @ nd.D + F @ nd.V.T
                if flops is not None:
                    m = nd.hi - nd.lo
                    flops.hss_mult += f_gemm(P, m, m) + f_gemm(P, F.shape[1], m)
            else:
                down = F @ nd.V.T
                if flops is not None:
                    flops.hss_mult += f_gemm(P, F.shape[1], nd.V.shape[0])
                cut = nodes[nd.left].V.shape[1]
                carry[nd.left], carry[nd.right] = down[:, :cut], down[:, cut:]
    return out


def hss_dense(T):
    """Dense reconstruction for testing (restates hss.py:364-394)."""
    if T.k > DENSE_LIMIT:
        raise ValueError("too large for dense reconstruction")
    return hss_apply_right(np.eye(T.k), T)


# ---------------------------------------------------------------------------
# merge-level update (dc.py:132-171)
# ---------------------------------------------------------------------------
@dataclass
class MergeInfo:
    size: int = 0
    kept: int = 0
    n_deflated: int = 0
    used_hss: bool = False
    hss_rank: int = 0
    fell_back: bool = False
    flops: dict = field(default_factory=dict)


def update_dense(Qb, G, flops=None):
    """dc.py:132-138 with the dense C from its generators."""
    Cd = G.dense(flops, "update_dense")
    if flops is not None:
        flops.update_dense += f_gemm(Qb.shape[0], *Cd.shape)
    return Qb @ Cd


def update_hss(Qb, G, leaf, oversample, rank_eps, rank_cap, seed, flops=None, info=None,
               Omega=None, return_tree=False, offdiag=False):
    """dc.py:141-171: partition, rank, construct, flag -> dense fallback, multiply."""
    def fallback():
        if info is not None:
            info.used_hss, info.fell_back = False, True
        out = update_dense(Qb, G, flops)
        return (out, None) if return_tree else out

    try:
        ranges = leaf_ranges(G.k, leaf, G.mu)
    except ValueError:
        return fallback()
    r = min(rank_estimate(ranges, G.d, G.gam, G.mu, rank_eps, rank_cap),
            min(hi - lo for lo, hi in ranges) - oversample)
    if r < 1:
        return fallback()
    T = rand_construct(G, ranges, r, oversample, seed, flops=flops, Omega=Omega, offdiag=offdiag)
    if T.flagged:
        return fallback()
    if info is not None:
        info.used_hss, info.hss_rank = True, T.r_used
    out = hss_apply_right(Qb, T, flops)
    return (out, T) if return_tree else out


# ---------------------------------------------------------------------------
# the rest of the DC recursion (dc.py:82-129, 174-257; secular.py:91-156)
# used for end-to-end parity of full eigendecompositions
# ---------------------------------------------------------------------------
def deflate(d, z, rho):
    """secular.py:91-156; returns (dk, zk, perm, rotations, defl_vals, n_defl)."""
    d = np.asarray(d, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = d.size
    tol = 8.0 * EPS * max(float(np.abs(d).max()), rho * float(np.sum(z * z)))
    order = np.argsort(d, kind="stable")
    ds, zs = d[order].copy(), z[order].copy()
    rots, keep, last = [], np.ones(n, dtype=bool), -1
    for t in range(n):
        if rho * abs(zs[t]) <= tol:
            keep[t] = False
            continue
        if last >= 0 and ds[t] - ds[last] <= tol:
            h = np.hypot(zs[last], zs[t])
            c, s = zs[last] / h, zs[t] / h
            zs[last], zs[t] = h, 0.0
            a, b = ds[last], ds[t]
            ds[last], ds[t] = c * c * a + s * s * b, s * s * a + c * c * b
            rots.append((int(order[last]), int(order[t]), float(c), float(s)))
            keep[t] = False
        else:
            last = t
    ki = np.flatnonzero(keep)
    di = np.flatnonzero(~keep)
    di = di[np.argsort(ds[di], kind="stable")]
    perm = np.concatenate([order[ki], order[di]]).astype(np.intp)
    return ds[ki], zs[ki], perm, rots, ds[di], di.size


@dataclass
class Config:
    """Mirror of SolverConfig (dc.py:30-51)."""
    base_size: int = 25
    hss_threshold: int = 2000
    leaf_size: int = 200
    oversample: int = 10
    rank_eps: float = 1e-16
    rank_cap: int = 100
    seed: int = 0
    method: str = "adc-rand"
    srrsc_tol: float = ID_TOL     # ADC1 only (srrsc_oracle.py)
    offdiag: bool = False         # the B200 path's off-diagonal sample (offdiag_samples)


def base_case(a, b):
    """dc.py:118-129"""
    n = a.size
    dd = a.copy()
    Q = np.eye(n)
    st = tql2(dd, b.copy(), Q, 30)
    if st != 0:
        raise BaseCaseError(f"QL iteration stalled on eigenvalue {st - 1}")
    o = np.argsort(dd, kind="stable")
    return dd[o], np.ascontiguousarray(Q[:, o])


def adc_solve(a, b, cfg=None):
    """Full DC eigendecomposition (dc.py:174-257). Returns (lam, Q, infos, flops)."""
    cfg = cfg or Config()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    flops = Flops()
    infos = []
    ids = itertools.count()

    def rec(a, b):
        n = a.size
        if n <= cfg.base_size:
            return base_case(a, b)
        h = n // 2
        bk = float(b[h - 1])
        rho = abs(bk)
        th = 1.0 if bk >= 0.0 else -1.0
        a1 = a[:h].copy(); a1[-1] -= rho
        a2 = a[h:].copy(); a2[0] -= rho
        L1, Q1 = rec(a1, b[:h - 1].copy())
        L2, Q2 = rec(a2, b[h:].copy())
        mid = next(ids)
        if rho == 0.0:
            dcat = np.concatenate([L1, L2])
            o = np.argsort(dcat, kind="stable")
            Q = np.zeros((n, n)); Q[:h, :h] = Q1; Q[h:, h:] = Q2
            return dcat[o], Q[:, o]
        zraw = np.concatenate([Q1[-1, :], th * Q2[0, :]]) / np.sqrt(2.0)
        dcat = np.concatenate([L1, L2])
        pm = np.argsort(dcat, kind="stable")
        dsrt, zsrt, reff = dcat[pm], zraw[pm], 2.0 * rho
        dk, zk, dperm, rots, ldef, nd = deflate(dsrt, zsrt, reff)
        k = dk.size
        info = MergeInfo(size=n, kept=k, n_deflated=nd)
        infos.append(info)
        before = flops.as_dict()
        Qb = np.zeros((n, n)); Qb[:h, :h] = Q1; Qb[h:, h:] = Q2
        for i, j, c, s in rots:
            ca, cb = Qb[:, pm[i]].copy(), Qb[:, pm[j]].copy()
            Qb[:, pm[i]] = c * ca + s * cb
            Qb[:, pm[j]] = -s * ca + c * cb
        ck, cd = pm[dperm[:k]], pm[dperm[k:]]
        if k > 0:
            G, lamk, _ = generators_from_roots(dk, zk, reff, flops)
            Qk = np.ascontiguousarray(Qb[:, ck])
            if cfg.method == "adc-rand" and k > cfg.hss_threshold:
                Qk = update_hss(Qk, G, cfg.leaf_size, cfg.oversample, cfg.rank_eps,
                                cfg.rank_cap, [cfg.seed, mid], flops, info,
                                offdiag=cfg.offdiag)
            elif cfg.method == "adc-srrsc" and k > cfg.hss_threshold:
                from .srrsc_oracle import update_srrsc
                Qk = update_srrsc(Qk, G, cfg.leaf_size, cfg.srrsc_tol, flops, info)
            else:
                Qk = update_dense(Qk, G, flops)
        else:
            Qk, lamk = np.zeros((n, 0)), np.zeros(0)
        info.flops = {p: v - before[p] for p, v in flops.as_dict().items()}
        lc = np.concatenate([lamk, ldef])
        Qc = np.hstack([Qk, Qb[:, cd]])
        o = np.argsort(lc, kind="stable")
        return lc[o], np.ascontiguousarray(Qc[:, o])

    lam, Q = rec(a, b)
    return lam, Q, infos, flops


# ---------------------------------------------------------------------------
# metrics (cli.py:63-71) and the BASELINE residual
# ---------------------------------------------------------------------------
def tridiag_dense(a, b):
    A = np.diag(a)
    i = np.arange(a.size - 1)
    A[i, i + 1] = b
    A[i + 1, i] = b
    return A


def norm_max(a, b):
    m = float(np.abs(a).max())
    return max(m, float(np.abs(b).max())) if b.size else m


def orthogonality(Q):
    n = Q.shape[0]
    return float(np.abs(Q.T @ Q - np.eye(n)).max()) / n


def backward(a, b, lam, Q):
    n = a.size
    return float(np.abs(tridiag_dense(a, b) - (Q * lam) @ Q.T).max()) / (norm_max(a, b) * n)


def residual(a, b, lam, Q):
    """||TQ - Q Lambda||_max / (N ||T||_max), O(N^2) for tridiagonal T."""
    TQ = a[:, None] * Q
    TQ[:-1] += b[:, None] * Q[1:]
    TQ[1:] += b[:, None] * Q[:-1]
    n = a.size
    return float(np.abs(TQ - Q * lam[None, :]).max()) / (n * norm_max(a, b))
