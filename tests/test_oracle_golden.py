"""Pin the CPU oracle (oracle/) against golden vectors from the unmodified reference."""
import numpy as np
import pytest

from helpers import EPS, align_columns, golden, unpack_tree
from oracle import hss_oracle as orc


@pytest.fixture(scope="module")
def sec():
    return golden("secular")


@pytest.fixture(scope="module")
def hssg():
    return golden("hss")


def test_secular_bit_exact_vs_reference(sec):
    # the C restatement follows _kernels.pyx:53-234 operation for operation
    for name in sec["names"]:
        d, z, rho = sec[f"{name}_d"], sec[f"{name}_z"], float(sec[f"{name}_rho"])
        lam, gam, mu, it = orc.secular_all(d, z, rho)
        np.testing.assert_array_equal(lam, sec[f"{name}_lam"])
        np.testing.assert_array_equal(gam, sec[f"{name}_gamma"])
        np.testing.assert_array_equal(mu, sec[f"{name}_mu"])
        assert it == int(sec[f"{name}_iters"])


def test_golden_ratio_roots():
    # pkg/tests/test_secular.py:106-109
    lam, _, _, _ = orc.secular_all(np.array([-1.0, 1.0]), np.array([1.0, 1.0]) / np.sqrt(2.0), 1.0)
    ref = np.array([(1 - np.sqrt(5)) / 2, (1 + np.sqrt(5)) / 2])
    np.testing.assert_allclose(lam, ref, rtol=1e-15)


def test_single_pole_exact():
    # pkg/tests/test_secular.py:98-103
    lam, gam, mu, it = orc.secular_all(np.array([0.7]), np.array([-0.3]), 2.0)
    assert lam[0] == 0.7 + 2.0 * 0.09 and gam[0] == 2.0 * 0.09 and mu[0] == 0.0 and it == 1


def test_loewner_and_normalizers_vs_reference(sec):
    for name in sec["names"]:
        if f"{name}_zhat" not in sec:
            continue
        d, z, rho = sec[f"{name}_d"], sec[f"{name}_z"], float(sec[f"{name}_rho"])
        gam, mu = sec[f"{name}_gamma"], sec[f"{name}_mu"]
        zh = orc.loewner(d, gam, mu, z, rho)
        np.testing.assert_allclose(zh, sec[f"{name}_zhat"], rtol=1e-13, atol=0)
        v = orc.normalizers(d, gam, mu, zh)
        np.testing.assert_allclose(v, sec[f"{name}_v"], rtol=1e-13, atol=0)


def test_secular_flop_counter(sec):
    for name in sec["names"]:
        d, z, rho = sec[f"{name}_d"], sec[f"{name}_z"], float(sec[f"{name}_rho"])
        f = orc.Flops()
        lam, gam, mu, _ = orc.solve_roots(d, z, rho, f)
        if d.size >= 2:
            zh = orc.loewner(d, gam, mu, z, rho, f)
            orc.normalizers(d, gam, mu, zh, f)
        assert f.secular == int(sec[f"{name}_flops_secular"])


def test_rank_bound_known_answer(hssg):
    assert orc.exp_sum_terms(2e3, 1e-13) == 33 == int(hssg["rank_bound_2e3_1e-13"])


@pytest.mark.parametrize("name", ["t256", "t600", "c4_2048"])
def test_hss_construction_vs_reference(hssg, name):
    g = hssg
    G = orc.Generators(g[f"{name}_d"], g[f"{name}_gamma"], g[f"{name}_mu"],
                       g[f"{name}_zhat"], g[f"{name}_v"])
    m = int(g[f"{name}_leaf"])
    ranges = orc.leaf_ranges(G.k, m, G.mu)
    assert [tuple(x) for x in g[f"{name}_ranges"]] == ranges
    r = min(orc.rank_estimate(ranges, G.d, G.gam, G.mu, float(g[f"{name}_eps"])),
            min(hi - lo for lo, hi in ranges) - 10)
    assert r == int(g[f"{name}_r"])
    seed = [int(s) for s in g[f"{name}_seed"]]
    Om = orc.sample_block(G.k, r + 10, seed)
    scale = np.abs(g[f"{name}_Y"]).max()
    assert np.abs(G.times(Om) - g[f"{name}_Y"]).max() <= 1e-13 * scale
    assert np.abs(G.t_times(Om) - g[f"{name}_Z"]).max() <= 1e-13 * np.abs(g[f"{name}_Z"]).max()
    f = orc.Flops()
    T = orc.rand_construct(G, ranges, r, 10, seed, flops=f)
    assert f.hss_construct == int(g[f"{name}_flops_construct"])
    assert T.r_used == int(g[f"{name}_tree_r_used"]) and int(T.flagged) == int(g[f"{name}_tree_flagged"])
    ref = unpack_tree(g, f"{name}_tree_")
    for nd, rn in zip(T.nodes, ref):
        assert (nd.lo, nd.hi, nd.level, nd.left, nd.right) == (rn["lo"], rn["hi"], rn["level"], rn["left"], rn["right"])
        if nd.U is not None:
            np.testing.assert_array_equal(nd.rsel, rn["rsel"])
            np.testing.assert_array_equal(nd.csel, rn["csel"])
            np.testing.assert_allclose(nd.U, rn["U"], atol=1e-10)
            np.testing.assert_allclose(nd.V, rn["V"], atol=1e-10)
        if nd.B is not None:
            np.testing.assert_allclose(nd.B.ravel(), rn["B"], rtol=1e-13, atol=1e-15)
    X = np.random.default_rng(99).standard_normal((40, G.k))
    f2 = orc.Flops()
    XH = orc.hss_apply_right(X, T, f2)
    assert f2.hss_mult == int(g[f"{name}_flops_mult"])
    assert np.abs(XH - g[f"{name}_XH"]).max() <= 1e-12 * np.abs(XH).max()
    Qold = np.random.default_rng(5).standard_normal((48, G.k))
    Qn = orc.update_hss(Qold, G, m, 10, float(g[f"{name}_eps"]), 100, seed)
    assert np.abs(Qn - g[f"{name}_Qnew"]).max() <= 1e-12 * np.abs(Qn).max()


def test_rank_starved_flags(hssg):
    g = hssg
    d, z, rho = g["starved_d"], g["starved_z"], float(g["starved_rho"])
    G, _, _ = orc.generators_from_roots(d, z, rho)
    T = orc.rand_construct(G, orc.leaf_ranges(256, 64, G.mu), 1, 0, 0)
    assert T.flagged == bool(g["starved_flagged"]) and len(T.flags) == int(g["starved_nflags"])


@pytest.mark.parametrize("fam", ["toeplitz", "kac", "uniform", "cfg5"])
@pytest.mark.parametrize("method", ["adc-rand", "dense-dc"])
def test_full_solve_vs_reference(fam, method):
    g = golden("adc")
    a, b = g[f"{fam}_a"], g[f"{fam}_b"]
    cfg = orc.Config(leaf_size=32, hss_threshold=128, rank_eps=1e-13, method=method)
    lam, Q, infos, fl = orc.adc_solve(a, b, cfg)
    tag = f"{fam}_{method}"
    nrm = orc.norm_max(a, b)
    assert np.abs(lam - g[f"{tag}_lam"]).max() <= 1e-12 * nrm
    got = np.array([[i.size, i.kept, i.n_deflated, int(i.used_hss), i.hss_rank, int(i.fell_back)]
                    for i in infos], dtype=np.int64)
    np.testing.assert_array_equal(got, g[f"{tag}_merges"])
    np.testing.assert_array_equal(np.array([fl.secular, fl.update_dense, fl.hss_construct, fl.hss_mult]),
                                  g[f"{tag}_flops"])
    assert orc.orthogonality(Q) <= 10 * max(float(g[f"{tag}_orth"]), EPS)
    assert orc.backward(a, b, lam, Q) <= 10 * max(float(g[f"{tag}_bwd"]), EPS)
    if fam in ("toeplitz", "kac"):   # well-separated spectra: columns comparable directly
        Qs = Q[:, ::8]
        assert np.abs(align_columns(Qs, g[f"{tag}_Qcols"]) - g[f"{tag}_Qcols"]).max() <= 1e-10
