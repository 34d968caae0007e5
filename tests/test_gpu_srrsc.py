"""ADC1 (SRRSC HSS construction, csrc/srrsc.cu) against its CPU definition
(oracle/srrsc_oracle.py; parity unpinned: the reference has no ADC1).

Pinned bit for bit: every node's rank, skeleton rows / columns (pivot order), saturation
flag, Schur residual and the leaf D / sibling B blocks.  To 1e-13: the interpolation bases
(their triangular solve sums in a different order).  End to end: ADC1 eigendecompositions
against the oracle's ADC1, dense DC and the closed forms."""
import ctypes

import numpy as np
import pytest
import torch

import paper_1510_04591_b200 as hb
from paper_1510_04591_b200 import _native
from paper_1510_04591_b200.flops import FlopCounter
from oracle import hss_oracle as orc
from oracle import srrsc_oracle as so

from helpers import config4_system

pytestmark = pytest.mark.gpu


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _system(kind, k, seed=0):
    if kind == "config4":
        d, u, rho = config4_system(k, seed)
    else:   # a Toeplitz-like merge: poles from the two halves of T(2, 1) interleaved
        h = k // 2
        l1 = np.sort(2 + 2 * np.cos(np.arange(1, h + 1) * np.pi / (h + 1)))
        l2 = np.sort(2 + 2 * np.cos(np.arange(1, k - h + 1) * np.pi / (k - h + 1)) + 1e-3)
        d = np.sort(np.concatenate([l1, l2]))
        u = np.random.default_rng(seed).standard_normal(k)
        u /= np.linalg.norm(u)
        rho = 1.0
    G, lam, _ = orc.generators_from_roots(d, u, rho)
    C = hb.CauchyEvecMatrix(G.d, G.gam, G.mu, G.zh, G.v)
    return G, C


@pytest.mark.parametrize("prune", ["0", "1"])
@pytest.mark.parametrize("kind,k,leaf", [("config4", 1024, 64), ("config4", 2048, 128),
                                         ("toeplitz", 1536, 48)])
def test_srrsc_tree_matches_definition(monkeypatch, kind, k, leaf, prune):
    # prune = "1": the block-pruned search (used from 12k columns off a node) forced on
    monkeypatch.setenv("HSSEIG_SRRSC_PRUNE", prune)
    G, C = _system(kind, k, seed=3)
    part = hb.build_partition(k, leaf, C.d, C.gamma, C.mu)
    ranges = orc.leaf_ranges(k, leaf, G.mu)
    assert list(part.ranges) == ranges
    cap = hb.srrsc_cap(part)
    assert cap == so.srrsc_cap(ranges)
    fo, fg = orc.Flops(), FlopCounter()
    ref = so.srrsc_construct(G, ranges, cap, 1e-15, fo)
    H = hb.srrsc_hss_construct(C, part, cap, tol=1e-15, flops=fg)
    assert H._status.read()[7] == 0     # the lazy search only ever read materialised blocks
    assert H.flagged == ref.flagged
    assert fg.hss_construct == fo.hss_construct
    rres = np_(H._view("rres", torch.float64, H.ct.n_nodes, 0))
    cres = np_(H._view("cres", torch.float64, H.ct.n_nodes, 0))
    for nd, rn in zip(H.nodes, ref.nodes):
        assert (nd.lo, nd.hi, nd.level) == (rn.lo, rn.hi, rn.level)
        if nd.index == H.root:
            continue
        np.testing.assert_array_equal(nd.rows_sel, rn.rsel)
        np.testing.assert_array_equal(nd.cols_sel, rn.csel)
        np.testing.assert_array_equal(nd.rows_local, rn.rloc)
        np.testing.assert_array_equal(nd.cols_local, rn.cloc)
        assert rres[nd.index] == rn.rres and cres[nd.index] == rn.cres
        np.testing.assert_allclose(nd.U, rn.U, rtol=0, atol=1e-13 * max(1.0, np.abs(rn.U).max()))
        np.testing.assert_allclose(nd.V, rn.V, rtol=0, atol=1e-13 * max(1.0, np.abs(rn.V).max()))
        np.testing.assert_array_equal(nd.B, rn.B)
        if nd.is_leaf:
            np.testing.assert_array_equal(nd.D, rn.D)
    A = np_(C.to_dense())
    dense = np_(hb.hss_to_dense(H))
    assert np.abs(dense - A).max() <= 1e-13
    X = np.random.default_rng(7).standard_normal((64, k))
    got = np_(hb.hss_matmul_right(X, H))
    want = orc.hss_apply_right(X, ref)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_srrsc_truncation_tolerance_orders_accuracy():
    G, C = _system("config4", 2048, seed=5)
    part = hb.build_partition(2048, 128, C.d, C.gamma, C.mu)
    A = C.to_dense()
    errs, ranks = [], []
    for tol in (1e-9, 1e-12, 1e-15):
        H = hb.srrsc_hss_construct(C, part, hb.srrsc_cap(part), tol=tol)
        errs.append(float((hb.hss_to_dense(H) - A).abs().max()))
        ranks.append(H.r_used)
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] <= 1e-14 and errs[0] <= 1e-8
    assert ranks[0] < ranks[1] < ranks[2]


def test_srrsc_saturation_flags_and_dense_fallback():
    G, C = _system("config4", 1024, seed=2)
    part = hb.build_partition(1024, 64, C.d, C.gamma, C.mu)
    H = hb.srrsc_hss_construct(C, part, 4, tol=1e-15)
    ref = so.srrsc_construct(G, orc.leaf_ranges(1024, 64, G.mu), 4, 1e-15)
    assert H.flagged and ref.flagged
    assert [(i, s) for i, s, _ in H.flags] == [(i, s) for i, s, _ in ref.flags]
    assert H.r_used == 4


def test_srrsc_argument_validation():
    G, C = _system("config4", 512, seed=1)
    part = hb.build_partition(512, 64, C.d, C.gamma, C.mu)
    with pytest.raises(ValueError):
        hb.srrsc_hss_construct(C, part, part.min_leaf + 1)
    with pytest.raises(ValueError):
        hb.srrsc_hss_construct(C, part, 0)
    with pytest.raises(ValueError):
        hb.srrsc_hss_construct(C, part, 8, tol=-1.0)
    with pytest.raises(ValueError):
        hb.SolverConfig(method="adc-srrsc", srrsc_tol=-1.0)


@pytest.mark.parametrize("nparts", [2, 4])
def test_srrsc_partitioned_levels_equal_single_build(nparts):
    from paper_1510_04591_b200.hss import HssTree, finish_construct
    from paper_1510_04591_b200.secular import Status
    G, C = _system("config4", 2048, seed=9)
    part = hb.build_partition(2048, 128, C.d, C.gamma, C.mu)
    cap = hb.srrsc_cap(part)
    H1 = hb.srrsc_hss_construct(C, part, cap)
    H2 = HssTree(part, cap)
    H2.method = "srrsc"
    lib = _native.load()
    work = torch.empty(int(lib.hsseig_srrsc_work_doubles(ctypes.byref(H2.ct))), dtype=torch.float64,
                       device="cuda")
    st = Status(2048)
    args = (C.gen, 1e-15, cap, ctypes.byref(H2.ct), _native.ptr(work), _native.ptr(st.t))
    s_lev = nparts.bit_length() - 1
    _native.check(lib.hsseig_tree_clear(ctypes.byref(H2.ct), _native.stream_ptr()), "clear")
    for p_ in range(nparts):
        _native.check(lib.hsseig_hss_build_srrsc_levels(*args, H2.ct.depth, s_lev, p_, nparts,
                                                        _native.stream_ptr()), "levels")
    _native.check(lib.hsseig_hss_build_srrsc_levels(*args, s_lev - 1, 0, 0, 1, _native.stream_ptr()),
                  "levels")
    H2._status = st
    finish_construct(H2)
    assert (H1.ranks()[0] == H2.ranks()[0]).all() and (H1.ranks()[1] == H2.ranks()[1]).all()
    X = torch.randn(100, 2048, dtype=torch.float64, device="cuda")
    assert torch.equal(hb.hss_matmul_right(X, H1), hb.hss_matmul_right(X, H2))


def _metrics(T, res):
    Q = res.Q
    n = T.n
    orth = float((Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max()) / n
    A = torch.as_tensor(T.to_dense(), device="cuda")
    lam = torch.as_tensor(res.lam, device="cuda")
    bwd = float((A - (Q * lam) @ Q.T).abs().max()) / (T.norm_max() * n)
    return orth, bwd


@pytest.mark.parametrize("fam", ["toeplitz", "kac", "uniform"])
def test_adc1_solve_matches_definition(fam):
    n = 1500
    if fam == "toeplitz":
        T = hb.gen_toeplitz(n)
    elif fam == "kac":
        T = hb.gen_kac(n)
    else:
        rng = np.random.default_rng(4)
        T = hb.SymTridiagonal(rng.uniform(-1, 1, n), rng.uniform(-1, 1, n - 1))
    cfg = hb.SolverConfig(leaf_size=48, hss_threshold=192, rank_eps=1e-13, method="adc-srrsc")
    res = hb.adc_solve(T, cfg)
    ocfg = orc.Config(leaf_size=48, hss_threshold=192, rank_eps=1e-13, method="adc-srrsc")
    lam_o, Q_o, infos, fl = orc.adc_solve(np.asarray(T.a), np.asarray(T.b), ocfg)
    nrm = T.norm_max()
    assert np.abs(res.lam - lam_o).max() <= 1e-12 * nrm
    got = [(m.size, m.kept, m.n_deflated, m.used_hss, m.hss_rank, m.fell_back) for m in res.merges]
    want = [(m.size, m.kept, m.n_deflated, m.used_hss, m.hss_rank, m.fell_back) for m in infos]
    assert got == want
    if fam != "uniform":
        assert any(m.used_hss for m in res.merges)
    orth, bwd = _metrics(T, res)
    eps = float(np.finfo(np.float64).eps)
    assert orth <= 10 * max(orc.orthogonality(Q_o), eps)
    assert bwd <= 10 * max(orc.backward(np.asarray(T.a), np.asarray(T.b), lam_o, Q_o), eps)


def test_adc1_toeplitz_closed_form_and_dense_dc():
    n = 3000
    T = hb.gen_toeplitz(n)
    res = hb.adc_solve(T, hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13,
                                          method="adc-srrsc"))
    ref = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.abs(res.lam - ref).max() <= 1e-12 * 4
    top = res.merges[-1]
    assert top.used_hss and not top.fell_back
    dd = hb.adc_solve(T, hb.SolverConfig(leaf_size=64, hss_threshold=256, method="dense-dc"))
    Qa = np_(res.Q)
    Qd = np_(dd.Q)
    s = np.sign((Qa * Qd).sum(axis=0))
    assert np.abs(Qa * s - Qd).max() <= 1e-10


def test_srrsc_pruned_search_equals_full_sweep_at_size(monkeypatch):
    # at a size where the pruned search is the default (k - |t| >= 12k columns): the tree is
    # bit-identical to the full sweep's (every pivot, rank, basis, flag)
    k = 24576
    d, u, rho = config4_system(k, 4)
    s = hb.RankOneSystem(d, u, rho)
    sol = hb.solve_secular(s)
    hb.recompute_weights(d, sol, u, rho=rho)
    C = hb.CauchyEvecMatrix.from_secular(s, sol)
    part = hb.build_partition(k, 128, C.d, C.gamma, C.mu)
    cap = hb.srrsc_cap(part)
    trees = []
    for prune in ("0", "1"):
        monkeypatch.setenv("HSSEIG_SRRSC_PRUNE", prune)
        trees.append(hb.srrsc_hss_construct(C, part, cap, tol=1e-15))
    A, B = trees
    assert B._status.read()[7] == 0
    assert A.flagged == B.flagged and A.r_used == B.r_used
    for na, nb in zip(A.nodes, B.nodes):
        if na.index == A.root:
            continue
        np.testing.assert_array_equal(na.rows_sel, nb.rows_sel)
        np.testing.assert_array_equal(na.cols_sel, nb.cols_sel)
        np.testing.assert_array_equal(np_(na.U), np_(nb.U))
        np.testing.assert_array_equal(np_(na.V), np_(nb.V))
        np.testing.assert_array_equal(np_(na.B), np_(nb.B))

