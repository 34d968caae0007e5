"""HSS approximation of the merge eigenvector matrix, built and applied on the GPU.

Host mirror of pkg/src/hsseig/hss.py.  Partition and rank estimate are O(#leaves)
host logic over a few pole gaps; the randomized construction (Algorithm 2) and
the structured product (Algorithm 3) run in libhsseig_b200.so
(csrc/hss_build.cu, csrc/hss_mult.cu).  The tree lives in one device blob laid
out by hsseig_tree_layout; per-node views are materialised only on request.
"""
import ctypes
import functools
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .flops import cauchy_eval_flops, cpqr_flops, gemm_flops
from .secular import Status, dev, dev_rows

DIST_SHIFT_THRESHOLD = 1e-10   # hss.py:20
MAX_BOUNDARY_SHIFT = 5         # hss.py:21
DEFAULT_RANK_CAP = 100         # hss.py:22
DEFAULT_ID_TOL = 1e-15         # hss.py:23
DENSE_BOUND = 4096             # hss.py:24
FLAG_TOL = 1e-12               # hss.py:117
MAX_WIDTH = 112                # sample width r + p supported by the sampling kernels


@dataclass(frozen=True)
class HssPartition:
    """Contiguous leaf ranges covering 0..k; power-of-two leaf count (hss.py:27-45)."""

    ranges: tuple
    leaf_size: int
    depth: int

    @property
    def k(self):
        return self.ranges[-1][1]

    @property
    def n_leaves(self):
        return len(self.ranges)

    @property
    def min_leaf(self):
        return min(hi - lo for lo, hi in self.ranges)

    def bounds(self):
        return np.array([lo for lo, _ in self.ranges] + [self.k], dtype=np.int32)


def _host(x):
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def build_partition(k, m, d=None, gamma=None, mu=None):
    """Near-equal power-of-two leaves; clustered boundaries slide up to 5 slots (hss.py:48-79)."""
    if k < 2 * m:
        raise ValueError(f"order {k} below twice the leaf size {m}")
    n_leaves = 1
    while n_leaves * m < k:
        n_leaves *= 2
    q, extra = divmod(k, n_leaves)
    starts = np.zeros(n_leaves + 1, dtype=np.int64)
    starts[1:] = np.cumsum([q + 1] * extra + [q] * (n_leaves - extra))
    mu = _host(mu)
    if mu is not None and n_leaves > 1:
        for b in range(1, n_leaves):
            s = int(starts[b])
            if mu[s - 1] >= DIST_SHIFT_THRESHOLD:
                continue
            cand = np.arange(max(starts[b - 1] + 1, s - MAX_BOUNDARY_SHIFT),
                             min(starts[b + 1] - 1, s + MAX_BOUNDARY_SHIFT) + 1)
            g = mu[cand - 1]
            if float(g.max()) > mu[s - 1]:
                starts[b] = cand[int(np.argmax(g))]
    ranges = tuple((int(starts[i]), int(starts[i + 1])) for i in range(n_leaves))
    return HssPartition(ranges=ranges, leaf_size=m, depth=int(math.log2(n_leaves)))


def rank_bound(R, eps):
    """Sum-of-exponentials term count for 1/x on [1, R] (hss.py:82-84)."""
    return int(math.ceil(math.log(16.0 / eps) * math.log(8.0 * R) / math.pi ** 2))


def estimate_rank(partition, d, gamma, mu, eps=1e-16, cap=DEFAULT_RANK_CAP):
    """Off-diagonal rank estimate from the boundary gaps (hss.py:87-103)."""
    if partition.n_leaves < 2:
        return 0
    starts = np.array([lo for lo, _ in partition.ranges[1:]], dtype=np.int64)
    if isinstance(mu, torch.Tensor):   # gather the few values needed on the device
        span = float((d[-1] + gamma[-1]) - d[0])
        dist = mu[torch.as_tensor(starts - 1, device=mu.device)].cpu().numpy()
    else:
        d, gamma, mu = _host(d), _host(gamma), _host(mu)
        span = (d[-1] + gamma[-1]) - d[0]
        dist = mu[starts - 1]
    r = 0
    for gap in dist:
        r = max(r, rank_bound(max(span / gap, 1.0), eps))
    return min(max(r, 1), cap)


class HssNode:
    """Host view of one tree node (hss.py:151-174); numeric fields download on demand."""

    def __init__(self, tree, index, level, lo, hi):
        self._t = tree
        self.index, self.level, self.lo, self.hi = index, level, lo, hi
        self.left = self.right = self.parent = self.sibling = -1

    @property
    def is_leaf(self):
        return self.left < 0

    def _rows(self, side):
        if self.index == self._t.root:
            return 0
        if self.is_leaf:
            return self.hi - self.lo
        r = self._t.ranks()[side]
        return int(r[self.left] + r[self.right])

    @property
    def U(self):
        if self.index == self._t.root:
            return None
        return self._t.slot("U", self.index, self._rows(0), int(self._t.ranks()[0][self.index]))

    @property
    def V(self):
        if self.index == self._t.root:
            return None
        return self._t.slot("V", self.index, self._rows(1), int(self._t.ranks()[1][self.index]))

    @property
    def B(self):
        if self.index == self._t.root:
            return None
        rU, rV = self._t.ranks()
        return self._t.slot("B", self.index, int(rU[self.index]), int(rV[self.sibling]))

    @property
    def D(self):
        if not self.is_leaf:
            return None
        return self._t.leaf_D(self.index)

    def _sel(self, name, side):
        if self.index == self._t.root:
            return None
        r = int(self._t.ranks()[side][self.index])
        return self._t.islot(name, self.index, r)

    rows_sel = property(lambda self: self._sel("rsel", 0))
    cols_sel = property(lambda self: self._sel("csel", 1))
    rows_local = property(lambda self: self._sel("rloc", 0))
    cols_local = property(lambda self: self._sel("cloc", 1))


@functools.lru_cache(maxsize=256)
def _topology(n_leaves):
    """Postorder structure of the balanced tree over n_leaves leaves (hss.py:188-214): children,
    parent, sibling (-1 where absent), level, first / last leaf of every node, position of a
    leaf among the leaves.  Depends on the leaf count only, so it is built once per count."""
    left, right, level, first, last = [], [], [], [], []

    def rec(a, b, lv):
        if b - a == 1:
            li = ri = -1
        else:
            h = (a + b) // 2
            li, ri = rec(a, h, lv + 1), rec(h, b, lv + 1)
        left.append(li)
        right.append(ri)
        level.append(lv)
        first.append(a)
        last.append(b - 1)
        return len(left) - 1

    rec(0, n_leaves, 0)
    left, right = np.array(left, dtype=np.int64), np.array(right, dtype=np.int64)
    n = len(left)
    parent, sib = np.full(n, -1, dtype=np.int64), np.full(n, -1, dtype=np.int64)
    inner = np.flatnonzero(left >= 0)
    parent[left[inner]] = parent[right[inner]] = inner
    sib[left[inner]], sib[right[inner]] = right[inner], left[inner]
    leaf = left < 0
    tp = {"leaf": leaf, "left": left, "right": right, "sib": sib, "parent": parent,
          "level": np.array(level, dtype=np.int64), "first": np.array(first, dtype=np.int64),
          "last": np.array(last, dtype=np.int64), "leaf_pos": np.cumsum(leaf) - 1}
    for v in tp.values():
        v.setflags(write=False)
    return tp


@dataclass
class HssTree:
    """Device-resident HSS tree (hss.py:177-185) with reference-compatible node views."""

    partition: HssPartition
    w: int
    k: int = 0
    r_used: int = 0
    flagged: bool = False
    flags: list = field(default_factory=list)
    seed: object = None

    def __post_init__(self):
        lib = nat.load()
        p = self.partition
        self.k = p.k
        self._bounds = p.bounds()
        mmax = int(np.diff(self._bounds).max())
        nbytes = int(lib.hsseig_tree_bytes(p.k, p.n_leaves, self.w, mmax))
        self.mem = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.ct = nat.Tree()
        b = np.ascontiguousarray(self._bounds, dtype=np.int32)
        nat.check(lib.hsseig_tree_layout(ctypes.byref(self.ct),
                                         b.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                         p.n_leaves, self.w, nat.ptr(self.mem), nat.stream_ptr()),
                  "tree_layout")
        self.root = int(self.ct.root)
        self._build_nodes()
        self._ranks = None

    # -- topology (postorder, identical to hss.py:188-214) --
    def _build_nodes(self):
        """Node arrays from the cached structure of a tree with this many leaves; the
        per-node HssNode views are only materialised on request (`nodes`): the solver's hot
        path (one tree per HSS merge) needs the arrays alone."""
        tp = _topology(self.partition.n_leaves)
        b = np.asarray(self._bounds, dtype=np.int64)
        lo, hi = b[tp["first"]], b[tp["last"] + 1]
        self._topo = dict(tp, lo=lo, hi=hi, m=hi - lo)
        self._leaf_pos = tp["leaf_pos"]
        self._nodes = None

    @property
    def nodes(self):
        if self._nodes is None:
            tp = self._topo
            nodes = []
            for i in range(len(tp["left"])):
                nd = HssNode(self, i, int(tp["level"][i]), int(tp["lo"][i]), int(tp["hi"][i]))
                nd.left, nd.right = int(tp["left"][i]), int(tp["right"][i])
                nd.parent, nd.sibling = int(tp["parent"][i]), int(tp["sib"][i])
                nodes.append(nd)
            self._nodes = nodes
        return self._nodes

    def levels(self):
        lv = self._topo["level"]
        return [np.flatnonzero(lv == l).tolist() for l in range(int(lv.max()) + 1)]

    # -- device views --
    def _view(self, attr, dtype, count, offset_elems):
        base = self.mem.data_ptr()
        off = getattr(self.ct, attr) - base
        esz = 8 if dtype == torch.float64 else 4
        start = off + offset_elems * esz
        return self.mem[start:start + count * esz].view(dtype)

    def ranks(self):
        if self._ranks is None:
            nn = self.ct.n_nodes
            rU = self._view("rU", torch.int32, nn, 0).cpu().numpy()
            rV = self._view("rV", torch.int32, nn, 0).cpu().numpy()
            self._ranks = (rU, rV)
        return self._ranks

    def slot(self, name, node, rows, cols):
        ws = self.ct.ws
        if name in ("U", "V"):   # candidate rows start at slot row 1 (row 0 is zero padding)
            n = self.ct.pmax * ws
            flat = self._view(name, torch.float64, n, node * n)
            return flat.view(-1, ws)[1:rows + 1, :cols].cpu().numpy().copy()
        n = ws * ws
        flat = self._view(name, torch.float64, n, node * n)
        return flat.view(-1, ws)[:rows, :cols].cpu().numpy().copy()

    def islot(self, name, node, r):
        ws = self.ct.ws
        return self._view(name, torch.int32, ws, node * ws)[:r].cpu().numpy().astype(np.intp)

    def leaf_D(self, node):
        mm = self.ct.dld
        drows = (self.ct.mmax + 1 + 15) // 16 * 16 + 2
        j = self._leaf_pos[node]
        n = drows * mm
        flat = self._view("D", torch.float64, n, j * n)
        m = int(self._topo["m"][node])
        return flat.view(drows, mm)[1:m + 1, :m].cpu().numpy().copy()


def tree_from_factors(partition, factors, w=None):
    """An HssTree holding given generators (the reference's HssNode fields, hss.py:151-185).

    factors maps a postorder node index to a dict with U, V (leaf: m x r, inner:
    (r_left + r_right) x r), B (r x r_sibling, every non-root node) and D (leaves, m x m).
    The slots are laid out exactly as the construction writes them, so the multiply and
    hss_to_dense run on it unchanged (used to test the multiply against closed forms).
    """
    ranks_u = {i: np.asarray(f["U"]).shape[1] for i, f in factors.items() if "U" in f}
    ranks_v = {i: np.asarray(f["V"]).shape[1] for i, f in factors.items() if "V" in f}
    rmax = max(list(ranks_u.values()) + list(ranks_v.values()) + [1])
    w = int(w or rmax)
    if w > partition.min_leaf or w > MAX_WIDTH:
        raise ValueError("ranks above the smallest leaf / supported width")
    tree = HssTree(partition, w)
    ct, nn = tree.ct, tree.ct.n_nodes
    lib = nat.load()
    nat.check(lib.hsseig_tree_clear(ctypes.byref(ct), nat.stream_ptr()), "tree_clear")
    ws, pmax = ct.ws, ct.pmax
    f64 = dict(dtype=torch.float64, device="cuda")
    rU = np.zeros(nn, dtype=np.int32)
    rV = np.zeros(nn, dtype=np.int32)
    for i in range(nn):
        rU[i] = ranks_u.get(i, 0)
        rV[i] = ranks_v.get(i, 0)
    tree._view("rU", torch.int32, nn, 0).copy_(torch.as_tensor(rU))
    tree._view("rV", torch.int32, nn, 0).copy_(torch.as_tensor(rV))
    Bv = tree._view("B", torch.float64, nn * ws * ws, 0).view(nn, ws, ws)
    Bv.zero_()
    drows = (ct.mmax + 1 + 15) // 16 * 16 + 2
    Dv = tree._view("D", torch.float64, partition.n_leaves * drows * ct.dld, 0).view(
        partition.n_leaves, drows, ct.dld)
    Dv.zero_()
    Uv = tree._view("U", torch.float64, nn * pmax * ws, 0).view(nn, pmax, ws)
    Vv = tree._view("V", torch.float64, nn * pmax * ws, 0).view(nn, pmax, ws)
    Vt = tree._view("Vt", torch.float64, nn * ws * pmax, 0).view(nn, ws, pmax)
    for nd in tree.nodes:
        i = nd.index
        f = factors.get(i, {})
        if i == tree.root:
            continue
        U = torch.as_tensor(np.asarray(f["U"], dtype=np.float64), **f64)
        V = torch.as_tensor(np.asarray(f["V"], dtype=np.float64), **f64)
        Uv[i, 1:1 + U.shape[0], :U.shape[1]] = U
        Vv[i, 1:1 + V.shape[0], :V.shape[1]] = V
        # V^T: candidate q at column q; an inner node's right-child candidates start at an
        # even column (16-byte TMA box starts)
        if nd.is_leaf:
            Vt[i, :V.shape[1], :V.shape[0]] = V.T
        else:
            na = int(rV[nd.left])
            sh = na & 1
            Vt[i, :V.shape[1], :na] = V[:na].T
            Vt[i, :V.shape[1], na + sh:V.shape[0] + sh] = V[na:].T
        B = torch.as_tensor(np.asarray(f["B"], dtype=np.float64), **f64)
        Bv[i, :B.shape[0], :B.shape[1]] = B
        if nd.is_leaf:
            D = torch.as_tensor(np.asarray(f["D"], dtype=np.float64), **f64)
            Dv[tree._leaf_pos[i], 1:1 + D.shape[0], :D.shape[1]] = D
    tree._ranks = None
    tree.r_used = int(max(rU.max(), rV.max()))
    tree.ct.rmax = tree.r_used
    return tree


def _construct_flops(tree, k, w):
    """hss_construct counter of hss.py:251-287 for the ranks the construction produced (the
    reference's per-node terms, summed over node arrays: a Python loop over the nodes cost
    ~10 ms per config-2 / config-3 solve)."""
    rU, rV = (np.asarray(r, dtype=np.int64) for r in tree.ranks())
    tp = tree._topo
    nonroot = np.ones(len(rU), dtype=bool)
    nonroot[tree.root] = False
    f = 2 * (gemm_flops(k, k, w) + cauchy_eval_flops(k * k))
    lf = tp["leaf"] & nonroot
    m = tp["m"][lf]
    f += int((6 * m * m + 2 * 2 * m * m * w + 4 * w * m * np.maximum(rU[lf], 1)
              + 4 * w * m * np.maximum(rV[lf], 1)).sum())
    inn = ~tp["leaf"]
    a, b = tp["left"][inn], tp["right"][inn]
    cross = 6 * (rU[a] * rV[b] + rU[b] * rV[a])          # B blocks of the children
    own = (2 * 2 * (rU[a] + rU[b]) * w * np.maximum(rU[a], rV[b])
           + 4 * w * (rU[a] + rU[b]) * np.maximum(rU[inn], 1)
           + 4 * w * (rV[a] + rV[b]) * np.maximum(rV[inn], 1))
    f += int(cross.sum()) + int(own[nonroot[inn]].sum())
    return f


def mult_flops(tree, P):
    """hss_mult counter of hss.py:329-357 for P rows."""
    rU, rV = (np.asarray(r, dtype=np.int64) for r in tree.ranks())
    tp = tree._topo
    nonroot = np.ones(len(rU), dtype=bool)
    nonroot[tree.root] = False
    lf = tp["leaf"] & nonroot
    m = tp["m"][lf]
    f = int((m * rU[lf] + m * m + rV[lf] * m).sum())
    inn = ~tp["leaf"] & nonroot
    a, b = tp["left"][inn], tp["right"][inn]
    f += int(((rU[a] + rU[b]) * rU[inn] + rV[inn] * (rV[a] + rV[b])).sum())
    f += int((rU[tp["sib"][nonroot]] * rV[nonroot]).sum())
    return 2 * P * f


FLAG_TOL = 1e-12   # hss.py:117


def _interp_rows(M, tol, max_rank):
    """Row ID with residual and saturation signal (hss.py:118-148), on the device.

    Returns (X, J, resid, saturated): X a CUDA tensor (p x r) with the identity on the rows
    J (NumPy intp), resid the trailing-mass estimate relative to ||M||_F.
    """
    Md = dev(M)
    if Md.ndim != 2:
        raise ValueError("M must be a matrix")
    p, w = Md.shape
    if p == 0 or w == 0 or max_rank == 0:
        return (torch.zeros(p, 0, dtype=torch.float64, device="cuda"), np.zeros(0, dtype=np.intp),
                0.0, False)
    lib = nat.load()
    if int(lib.hsseig_interp_smem_bytes(p, w)) > 227 * 1024:
        raise ValueError(f"{p} x {w} is too large for one shared-memory ID")
    Md = Md.contiguous()
    mr = int(max_rank)
    X = torch.zeros(p, max(mr, 1), dtype=torch.float64, device="cuda")
    J = torch.zeros(max(mr, 1), dtype=torch.int32, device="cuda")
    rk = torch.zeros(1, dtype=torch.int32, device="cuda")
    rs = torch.zeros(1, dtype=torch.float64, device="cuda")
    sat = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.hsseig_interp_decomp(nat.ptr(Md), Md.stride(0), 0, p, w, 1, float(tol), mr,
                                       nat.ptr(X), X.stride(0), 0, nat.ptr(J), nat.ptr(rk),
                                       nat.ptr(rs), nat.ptr(sat), nat.stream_ptr()), "interp_decomp")
    r = int(rk.cpu()[0])
    return (X[:, :r], J[:r].cpu().numpy().astype(np.intp), float(rs.cpu()[0]), bool(int(sat.cpu()[0])))


def interpolative_decomp(M, tol, max_rank):
    """Row interpolative decomposition M ~= X @ M[J, :] (hss.py:104-111)."""
    X, J, _, _ = _interp_rows(M, tol, max_rank)
    return X, J


def sample_omega(k, w, seed):
    """The reference's Gaussian sample block (hss.py:236-237), drawn on the host."""
    return np.random.default_rng(seed).standard_normal((k, w))


_STREAM = {"ns": None}


def draw_omega(k, w, seed):
    """default_rng(seed).standard_normal((k, w)) on the device, bit-identical to the host
    draw (csrc/normals.cu, checked against NumPy once per process); rows padded to an even
    leading dimension for the TMA sampler.  Falls back to the host draw only when NumPy's
    ziggurat tables cannot be located."""
    from . import sample_rng
    if not sample_rng.available():
        return dev(sample_omega(k, w, seed))
    n = k * w
    ns = _STREAM["ns"]
    if ns is None or ns.nmax < n:
        ns = _STREAM["ns"] = sample_rng.NormalStream(n)
    ld = w + (w & 1)
    om = torch.empty(k, ld, dtype=torch.float64, device="cuda")
    if ld != w:
        om[:, w:] = 0.0
    ns.draw(seed, n, om, w=w, ld=ld)
    ns.fixup()
    return om[:, :w]


def draw_omegas(specs, streams=None):
    """draw_omega for several (k, w, seed) at once: every draw is enqueued first (draw i on
    streams[i] when given), then one wait per draw covers its tail read-back."""
    from . import sample_rng
    cur = torch.cuda.current_stream()
    st = [streams[i] if streams else cur for i in range(len(specs))]
    if not sample_rng.available():
        out = []
        for (k, w, seed), s in zip(specs, st):
            with torch.cuda.stream(s):
                out.append(draw_omega(k, w, seed))
        return out
    pool = _STREAM.setdefault("pool", [])
    out = []
    for i, (k, w, seed) in enumerate(specs):
        n = k * w
        if i == len(pool):
            pool.append(None)
        if pool[i] is None or pool[i].nmax < n:
            pool[i] = None
            pool[i] = sample_rng.NormalStream(n)
        ld = w + (w & 1)
        with torch.cuda.stream(st[i]):
            om = torch.empty(k, ld, dtype=torch.float64, device="cuda")
            if ld != w:
                om[:, w:] = 0.0
            pool[i].draw(seed, n, om, w=w, ld=ld)
        out.append(om[:, :w])
    for i in range(len(specs)):
        with torch.cuda.stream(st[i]):
            pool[i].fixup()
    return out


def rand_hss_construct(A, partition, r, p=10, seed=0, id_tol=DEFAULT_ID_TOL, flops=None,
                       omega=None, finish=True, offdiag=True):
    """Randomized bottom-up construction from one Gaussian sample (hss.py:217-306).

    offdiag (default): the leaves' Phi / Theta come from the off-diagonal sample
    C(t, t^c) Omega(t^c) instead of Y_t - D_t Omega_t (hss.py:265-266); mathematically the
    same matrices, without the cancellation that leaves the sample's rounding noise for the
    ID to truncate against.  offdiag=False is the reference's arithmetic."""
    if partition.n_leaves < 2:
        raise ValueError("need at least two leaves; use the dense path instead")
    if r < 1 or p < 0:
        raise ValueError("need rank estimate >= 1 and oversampling >= 0")
    w = r + p
    if w > partition.min_leaf:
        raise ValueError(f"sample width {w} exceeds smallest leaf {partition.min_leaf}")
    if w > MAX_WIDTH:
        raise ValueError(f"sample width {w} above the supported {MAX_WIDTH}")
    om = dev(omega) if omega is not None else draw_omega(A.k, w, seed)
    tree = HssTree(partition, w, seed=seed)
    tree.offdiag = bool(offdiag)
    Y, Z = A.sample(om, leaf_of=tree.ct.leaf_of if offdiag else None)
    st = Status(A.k)
    nat.check(nat.load().hsseig_hss_build_rand(A.gen, nat.ptr(om), om.stride(0), nat.ptr(Y),
                                               nat.ptr(Z), Y.stride(0), float(id_tol),
                                               int(bool(offdiag)), ctypes.byref(tree.ct),
                                               nat.ptr(st.t), nat.stream_ptr()), "hss_build_rand")
    tree._status = st
    tree._omega = om
    if finish:
        finish_construct(tree, flops)
    return tree


def srrsc_hss_construct(A, partition, cap, tol=DEFAULT_ID_TOL, flops=None, finish=True, work=None):
    """ADC1: HSS tree of C from its generators by structured rank-revealing Schur complements.

    No reference implementation exists; the definition is
    oracle/srrsc_oracle.py (parity unpinned).  cap is the largest node rank (tree width);
    the tree has the layout of rand_hss_construct, so finish_construct / hss_matmul_right /
    hss_to_dense apply to it unchanged.  Replaces the construction call of dc.py:165.
    """
    if partition.n_leaves < 2:
        raise ValueError("need at least two leaves; use the dense path instead")
    if cap < 1 or cap > partition.min_leaf or cap > MAX_WIDTH:
        raise ValueError(f"rank cap {cap} outside [1, min(smallest leaf, {MAX_WIDTH})]")
    if not tol >= 0.0:
        raise ValueError("tolerance must be non-negative")
    tree = HssTree(partition, cap)
    tree.method = "srrsc"
    lib = nat.load()
    nw = int(lib.hsseig_srrsc_work_doubles(ctypes.byref(tree.ct)))
    if work is None or work.numel() < nw:
        work = torch.empty(nw, dtype=torch.float64, device="cuda")
    st = Status(A.k)
    nat.check(lib.hsseig_hss_build_srrsc(A.gen, float(tol), int(cap), ctypes.byref(tree.ct),
                                         nat.ptr(work), nat.ptr(st.t), nat.stream_ptr()),
              "hss_build_srrsc")
    tree._status = st
    tree._work = work      # alive until the queued construction has run
    if finish:
        finish_construct(tree, flops)
    return tree


def _srrsc_flops(tree, k):
    """Construction counter of oracle/srrsc_oracle.py: every elimination sweep evaluates the
    whole candidate block (6 per entry, cauchy.py:55 convention), p r^2 for the bases, and the
    D / B entries.  Summed over node arrays (see _construct_flops)."""
    rU, rV = (np.asarray(r, dtype=np.int64) for r in tree.ranks())
    tp = tree._topo
    nonroot = np.ones(len(rU), dtype=bool)
    nonroot[tree.root] = False
    inn = ~tp["leaf"]
    a, b = tp["left"][inn], tp["right"][inn]
    f = int((6 * (rU[a] * rV[b] + rU[b] * rV[a])).sum())      # B blocks, the root's included
    lf = tp["leaf"] & nonroot
    f += int((6 * tp["m"][lf] * tp["m"][lf]).sum())            # D blocks
    # candidate counts of the two sides: a leaf's own indices, an inner node's children's skeletons
    pU, pV = tp["m"].copy(), tp["m"].copy()
    pU[inn], pV[inn] = rU[a] + rU[b], rV[a] + rV[b]
    ncomp = k - tp["m"]
    for pc, r in ((pU, rU), (pV, rV)):
        f += int((6 * (r + 1) * pc * ncomp + pc * r * r)[nonroot].sum())
    return f


def _construct_parts(tree):
    nn = tree.ct.n_nodes
    parts = [tree._view("rres", torch.float64, nn, 0), tree._view("cres", torch.float64, nn, 0),
             tree._view("flags", torch.int32, 2 * nn, 0), tree._view("rU", torch.int32, nn, 0),
             tree._view("rV", torch.int32, nn, 0)]
    return torch.cat([t.view(torch.uint8) for t in parts])


def prefetch_construct(tree, extra=None):
    """Queue the host read-back finish_construct needs (flags, residuals, ranks; plus
    `extra` = (device tensor, pinned host tensor) pairs) as pinned async copies behind the
    construction, so later work (the multiply) can be queued before the host waits.
    Returns the handle for finish_construct(pre=...)."""
    dev = _construct_parts(tree)
    buf = getattr(tree, "_host_blob", None)
    if buf is None or buf.numel() != dev.numel():
        buf = tree._host_blob = torch.empty(dev.numel(), dtype=torch.uint8, pin_memory=True)
    buf.copy_(dev, non_blocking=True)
    for d, h in (extra or ()):
        h.copy_(d, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return buf, ev


def finish_construct(tree, flops=None, pre=None):
    """Host read-back after construction: flags, ranks, r_used and the flop counter.
    pre: the handle of prefetch_construct (waits for that read-back only, not the stream)."""
    nn = tree.ct.n_nodes
    # one read-back for flags, residuals and ranks
    if pre is None:
        blob = _construct_parts(tree).cpu().numpy()
        tree._status.read()
    else:
        pre[1].synchronize()
        blob = pre[0].numpy()
    rr = blob[:8 * nn].view(np.float64)
    cr = blob[8 * nn:16 * nn].view(np.float64)
    fl = blob[16 * nn:24 * nn].view(np.int32).reshape(nn, 2)
    tree._ranks = (blob[24 * nn:28 * nn].view(np.int32).copy(), blob[28 * nn:32 * nn].view(np.int32).copy())
    tree.flags = []
    # the reference appends flags in processing order: deepest level first, postorder within
    flagged = np.flatnonzero(fl.any(axis=1))
    flagged = flagged[flagged != tree.root]
    for idx in sorted(flagged.tolist(), key=lambda i: -int(tree._topo["level"][i])):
        if fl[idx, 0]:
            tree.flags.append((idx, "row", float(rr[idx])))
        if fl[idx, 1]:
            tree.flags.append((idx, "col", float(cr[idx])))
    tree.flagged = bool(fl.any())        # per-node saturation flags (also right after a gather)
    rU, rV = tree.ranks()
    mask = np.ones(nn, dtype=bool)
    mask[tree.root] = False
    tree.r_used = int(max(rU[mask].max(), rV[mask].max()))
    tree.ct.rmax = tree.r_used      # the multiply sizes its output tiles to the ranks
    if flops is not None:
        if getattr(tree, "method", "rand") == "srrsc":
            flops.hss_construct += _srrsc_flops(tree, tree.k)
        else:
            flops.hss_construct += _construct_flops(tree, tree.k, tree.w)
    return tree


MULT_WORK_BUDGET = int(float(os.environ.get("HSSEIG_MULT_WORK_GB", "16")) * (1 << 30))


def hss_matmul_right(X, H, flops=None, out=None):
    """Structured product X @ H (hss.py:309-361) as per-level batched DMMA GEMMs."""
    X = dev_rows(X)
    if X.ndim == 1:
        X = X[None, :]
    if X.shape[1] != H.k:
        raise ValueError(f"X has {X.shape[1]} columns, tree order is {H.k}")
    if X.stride(0) % 2 or X.data_ptr() % 16:   # TMA reads X with 16-byte aligned rows
        Xp = torch.empty(X.shape[0], X.shape[1] + (X.shape[1] & 1), dtype=torch.float64, device="cuda")
        Xp[:, :X.shape[1]] = X
        X = Xp[:, :X.shape[1]]
    P = X.shape[0]
    lib = nat.load()
    if out is None:
        out = torch.empty(P, H.k, dtype=torch.float64, device="cuda")
    # the per-level G/F workspace grows with the rows: bound it by multiplying row chunks
    base = int(lib.hsseig_matmul_work_doubles(0, ctypes.byref(H.ct)))
    per_row = int(lib.hsseig_matmul_work_doubles(1, ctypes.byref(H.ct))) - base
    chunk = max(128, (MULT_WORK_BUDGET // 8 - base) // max(per_row, 1) // 128 * 128)
    chunk = min(chunk, P)
    work = torch.empty(base + per_row * chunk, dtype=torch.float64, device="cuda")
    for r0 in range(0, P, chunk):
        r1 = min(P, r0 + chunk)
        nat.check(lib.hsseig_hss_matmul_right(nat.ptr(X[r0:r1]), X.stride(0), r1 - r0,
                                              ctypes.byref(H.ct), nat.ptr(out[r0:r1]),
                                              out.stride(0), nat.ptr(work), nat.stream_ptr()),
                  "hss_matmul_right")
    if flops is not None:
        flops.hss_mult += mult_flops(H, P)
    return out


def hss_to_dense(H, bound=DENSE_BOUND):
    """Dense reconstruction (testing utility, hss.py:375-394) via the identity probe."""
    if H.k > bound:
        raise ValueError(f"order {H.k} above the dense reconstruction bound {bound}")
    return hss_matmul_right(torch.eye(H.k, dtype=torch.float64, device="cuda"), H)


def audit_tree(H):
    """Structural invariants of a constructed tree (hss.py:397-431); AssertionError on failure.

    Postorder topology, children tiling their parent, contiguous leaves, and the identity
    rows of every interpolation basis at its skeleton (U[rows_local] = I, V[cols_local] = I)
    read back from the device slots."""
    nodes = H.nodes
    root = nodes[H.root]
    assert H.root == len(nodes) - 1, "root must be last in postorder"
    leaves = []
    for nd in nodes:
        if nd.is_leaf:
            leaves.append(nd)
            continue
        lt, rt = nodes[nd.left], nodes[nd.right]
        assert nd.left < nd.right < nd.index, f"postorder violated at {nd.index}"
        assert lt.parent == nd.index and rt.parent == nd.index
        assert lt.sibling == nd.right and rt.sibling == nd.left
        assert (lt.lo, rt.hi) == (nd.lo, nd.hi) and lt.hi == rt.lo, \
            f"children ranges must tile node {nd.index}"
        assert lt.level == rt.level == nd.level + 1
    leaves.sort(key=lambda n: n.lo)
    assert leaves[0].lo == 0 and leaves[-1].hi == H.k
    for a, b in zip(leaves, leaves[1:]):
        assert a.hi == b.lo, "leaf ranges must be contiguous"
    assert (root.lo, root.hi) == (0, H.k)
    for nd in nodes:
        if nd.index == H.root:
            continue
        U, V = nd.U, nd.V
        assert np.array_equal(U[nd.rows_local], np.eye(U.shape[1])), \
            f"U of node {nd.index} lost its identity submatrix"
        assert np.array_equal(V[nd.cols_local], np.eye(V.shape[1])), \
            f"V of node {nd.index} lost its identity submatrix"
        rs, cs = nd.rows_sel, nd.cols_sel
        if rs.size:
            assert nd.lo <= rs.min() and rs.max() < nd.hi
        if cs.size:
            assert nd.lo <= cs.min() and cs.max() < nd.hi
