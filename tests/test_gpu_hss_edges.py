"""HSS construction / multiply edge cases (mirrors pkg/tests/test_hss.py): generator-held
trees against the closed-form dense matrix, zero couplings, support confined to one
leaf, seed determinism, argument validation, shape errors, flop scaling, orthogonality."""
import numpy as np
import pytest
import scipy.linalg
import torch

import paper_1510_04591_b200 as hb
from paper_1510_04591_b200 import hss
from paper_1510_04591_b200.flops import FlopCounter

from helpers import random_system

pytestmark = pytest.mark.gpu


def _manual(rng, n_leaves, leaf, rank):
    part = hb.build_partition(n_leaves * leaf, leaf)
    probe = hss.HssTree(part, rank)
    factors = {}
    for nd in probe.nodes:
        f = {}
        if nd.index != probe.root:
            rows = leaf if nd.is_leaf else 2 * rank
            f["U"] = rng.standard_normal((rows, rank))
            f["V"] = rng.standard_normal((rows, rank))
            f["B"] = rng.standard_normal((rank, rank))
        if nd.is_leaf:
            f["D"] = rng.standard_normal((leaf, leaf))
        factors[nd.index] = f
    return hss.tree_from_factors(part, factors), factors, probe


def test_to_dense_two_leaf_formula():
    rng = np.random.default_rng(31)
    tree, f, probe = _manual(rng, 2, 6, 2)
    l, r = f[0], f[1]
    expect = np.block([[l["D"], l["U"] @ l["B"] @ r["V"].T],
                       [r["U"] @ r["B"] @ l["V"].T, r["D"]]])
    np.testing.assert_allclose(hb.hss_to_dense(tree).cpu().numpy(), expect, atol=1e-14)


def test_to_dense_four_leaf_nesting():
    rng = np.random.default_rng(32)
    tree, f, _ = _manual(rng, 4, 5, 2)
    n1, n2, n3, n4, n5, n6 = (f[i] for i in range(6))
    ul = np.block([[n1["D"], n1["U"] @ n1["B"] @ n2["V"].T], [n2["U"] @ n2["B"] @ n1["V"].T, n2["D"]]])
    lr = np.block([[n4["D"], n4["U"] @ n4["B"] @ n5["V"].T], [n5["U"] @ n5["B"] @ n4["V"].T, n5["D"]]])
    U3 = scipy.linalg.block_diag(n1["U"], n2["U"]) @ n3["U"]
    V3 = scipy.linalg.block_diag(n1["V"], n2["V"]) @ n3["V"]
    U6 = scipy.linalg.block_diag(n4["U"], n5["U"]) @ n6["U"]
    V6 = scipy.linalg.block_diag(n4["V"], n5["V"]) @ n6["V"]
    expect = np.block([[ul, U3 @ n3["B"] @ V6.T], [U6 @ n6["B"] @ V3.T, lr]])
    np.testing.assert_allclose(hb.hss_to_dense(tree).cpu().numpy(), expect, atol=1e-13)


def test_matmul_blockdiag_when_b_zero():
    rng = np.random.default_rng(33)
    tree, f, probe = _manual(rng, 4, 32, 5)
    for i in f:
        if "B" in f[i]:
            f[i]["B"] = np.zeros_like(f[i]["B"])
    tree = hss.tree_from_factors(tree.partition, f)
    X = rng.standard_normal((5, 128))
    out = hb.hss_matmul_right(X, tree).cpu().numpy()
    ref = np.zeros_like(out)
    for nd in probe.nodes:
        if nd.is_leaf:
            ref[:, nd.lo:nd.hi] = X[:, nd.lo:nd.hi] @ f[nd.index]["D"]
    np.testing.assert_allclose(out, ref, atol=1e-15)


def _cauchy(rng, k):
    d, z, rho = random_system(rng, k)
    rs = hb.RankOneSystem(d, z, rho)
    sol = hb.solve_secular(rs)
    hb.recompute_weights(rs.d, sol, rs.z, rho=rho)
    return hb.CauchyEvecMatrix.from_secular(rs, sol)


def _built(rng, k, m=64, seed=0):
    C = _cauchy(rng, k)
    part = hb.build_partition(k, m, C.d, C.gamma, C.mu)
    r = min(hb.estimate_rank(part, C.d, C.gamma, C.mu, 1e-13), part.min_leaf - 10)
    return C, part, hb.rand_hss_construct(C, part, r, p=10, seed=seed), r


def test_construct_support_confined_to_first_leaf():
    rng = np.random.default_rng(34)
    k = 128
    zhat = np.zeros(k)
    v = np.zeros(k)
    zhat[:32] = rng.standard_normal(32)
    v[:32] = rng.standard_normal(32)
    C = hb.CauchyEvecMatrix(np.arange(1.0, k + 1.0), np.full(k, 0.3), np.full(k, 0.7), zhat, v)
    part = hb.build_partition(k, 32)
    H = hb.rand_hss_construct(C, part, r=8, p=8, seed=3)
    dense = hb.hss_to_dense(H).cpu().numpy()
    A = C.to_dense().cpu().numpy()
    scale = np.abs(A).max()
    for nd in H.nodes:
        B = nd.B
        if B is not None and B.size:
            assert np.abs(B).max() <= 1e-12 * scale
    off = dense.copy()
    off[:32, :32] = 0.0
    assert np.abs(off).max() <= 1e-12 * scale
    assert np.abs(dense - A).max() <= 1e-12 * scale


def test_construct_deterministic_in_seed():
    C, part, H1, r = _built(np.random.default_rng(35), 256, seed=11)
    H2 = hb.rand_hss_construct(C, part, r, p=10, seed=11)
    for a, b in zip(H1.nodes, H2.nodes):
        if a.U is not None:
            np.testing.assert_array_equal(a.U, b.U)
        if a.B is not None:
            np.testing.assert_array_equal(a.B, b.B)


def test_construct_validates_inputs():
    C, part, _, _ = _built(np.random.default_rng(36), 256)
    with pytest.raises(ValueError):
        hb.rand_hss_construct(C, part, r=0, p=10)
    with pytest.raises(ValueError):
        hb.rand_hss_construct(C, part, r=60, p=10)   # r + p above the smallest leaf


def test_matmul_shape_mismatch():
    _, _, H, _ = _built(np.random.default_rng(37), 256)
    with pytest.raises(ValueError):
        hb.hss_matmul_right(np.zeros((3, 255)), H)


def test_to_dense_respects_bound():
    _, _, H, _ = _built(np.random.default_rng(38), 256)
    with pytest.raises(ValueError):
        hb.hss_to_dense(H, bound=100)


def test_matmul_flop_scaling():
    rng = np.random.default_rng(39)
    totals = {}
    for k in (512, 1024, 2048):
        C = _cauchy(rng, k)
        part = hb.build_partition(k, 64, C.d, C.gamma, C.mu)
        H = hb.rand_hss_construct(C, part, r=30, p=10, seed=5)
        f = FlopCounter()
        hb.hss_matmul_right(torch.eye(k, dtype=torch.float64, device="cuda"), H, flops=f)
        totals[k] = f.hss_mult
    assert totals[1024] / totals[512] <= 5.0
    assert totals[2048] / totals[1024] <= 5.0


def test_orthogonality_preserved_through_compression():
    C, part, H, _ = _built(np.random.default_rng(40), 512, seed=2)
    A = C.to_dense()
    dense = hb.hss_to_dense(H)
    delta = float(torch.linalg.norm(dense - A))
    I = torch.eye(512, dtype=torch.float64, device="cuda")
    assert float((dense.T @ dense - I).abs().max()) <= 3 * delta
