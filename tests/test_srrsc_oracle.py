"""CPU checks of the ADC1 definition (oracle/srrsc_oracle.py; parity unpinned):
the generator recurrence reproduces the explicit Schur complement, the stable eigenvalue
differences, the HSS reconstruction error follows the tolerance, and full ADC1 solves meet
the closed forms.  These pin the checker the GPU tests (test_gpu_srrsc.py) compare against."""
import numpy as np
import pytest

from oracle import hss_oracle as orc
from oracle import srrsc_oracle as so

from helpers import config4_system


def _gen(k, seed):
    d, u, rho = config4_system(k, seed)
    G, lam, _ = orc.generators_from_roots(d, u, rho)
    return G, lam


def test_lamdiff_is_the_eigenvalue_difference():
    G, lam = _gen(600, 1)
    rng = np.random.default_rng(0)
    a = rng.integers(0, 600, 2000)
    b = rng.integers(0, 600, 2000)
    got = so.lamdiff(G, a, b)
    want = lam[a] - lam[b]
    assert np.all(got[a == b] == 0.0)
    # no cancellation: relative accuracy even for neighbouring roots
    m = a != b
    assert np.all(np.abs(got[m] - want[m]) <= 1e-12 * np.abs(want[m]) + 4e-16)
    assert np.all(np.sign(got[m]) == np.sign(want[m]))


@pytest.mark.parametrize("side", ["row", "col"])
def test_generator_recurrence_is_the_schur_complement(side):
    # with a loose tolerance the residual sits far above rounding: the ID error
    # M - X M[J] is then exactly the Schur complement the recurrence left behind
    G, _ = _gen(768, 2)
    C = G.dense()
    lo, hi = 256, 384
    cand = np.arange(lo, hi)
    comp = np.r_[0:lo, hi:768]
    M = C[np.ix_(cand, comp)] if side == "row" else C[np.ix_(comp, cand)].T
    X, J, res, sat, r = so.srrsc_block(G, cand, lo, hi, side, 1e-7, 64)
    assert 0 < r < 64 and not sat
    np.testing.assert_array_equal(X[J], np.eye(r))
    err = np.abs(M - X @ M[J]).max() / np.abs(M).max()
    assert res <= 1e-7
    assert abs(err - res) <= 1e-4 * res
    # complete pivoting: the first pivot is the block's largest entry
    assert np.abs(M[J[0]]).max() == np.abs(M).max()


def test_construct_reconstruction_follows_tolerance():
    G, _ = _gen(1024, 3)
    C = G.dense()
    ranges = orc.leaf_ranges(1024, 64, G.mu)
    prev = None
    for tol in (1e-8, 1e-12, 1e-15):
        T = so.srrsc_construct(G, ranges, so.srrsc_cap(ranges), tol)
        assert not T.flagged
        err = np.abs(orc.hss_dense(T) - C).max()
        assert err <= 50 * tol
        if prev is not None:
            assert T.r_used >= prev
        prev = T.r_used
    assert prev < 64          # compressed: ranks below the leaf size


def test_oracle_adc1_toeplitz_closed_form():
    n = 1200
    a, b = np.full(n, 2.0), np.ones(n - 1)
    cfg = orc.Config(leaf_size=48, hss_threshold=192, rank_eps=1e-13, method="adc-srrsc")
    lam, Q, infos, fl = orc.adc_solve(a, b, cfg)
    ref = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.abs(lam - ref).max() <= 1e-12 * 4
    assert any(i.used_hss for i in infos)
    assert orc.orthogonality(Q) <= 1e-16
    assert orc.residual(a, b, lam, Q) <= 1e-16
    assert fl.hss_construct > 0
