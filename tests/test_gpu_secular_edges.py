"""Secular / Loewner / stable-gap identities (mirrors pkg/tests/test_secular.py) on the GPU
kernels: interlacing and gap-pair identities, the residual bound, weight hand cases and
sign convention, stable-gap branches, small-system eigenvector orthogonality."""
import numpy as np
import pytest
import torch

import paper_1510_04591_b200 as hb
from paper_1510_04591_b200.secular import gap_table, stable_gap

from helpers import EPS, random_system

pytestmark = pytest.mark.gpu


def _solve(d, z, rho):
    sys = hb.RankOneSystem(d, z, rho)
    sol = hb.solve_secular(sys)
    return sys, sol


def _np(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _golden():
    return np.array([-1.0, 1.0]), np.array([1.0, 1.0]) / np.sqrt(2.0), 1.0


@pytest.mark.parametrize("k", [2, 7, 33])
def test_interlacing_and_gap_identities(k):
    d, z, rho = random_system(np.random.default_rng(k), k)
    sys, sol = _solve(d, z, rho)
    lam, gam, mu = _np(sol.lam), _np(sol.gamma), _np(sol.mu)
    assert np.all(lam > d) and np.all(lam[:-1] < d[1:])
    assert lam[-1] < d[-1] + rho * np.sum(z ** 2)
    assert np.all(gam > 0) and np.all(mu[:-1] > 0) and mu[-1] >= 0
    np.testing.assert_allclose(d + gam, lam, rtol=1e-15)
    dnext = np.append(d[1:], sol.pole_bound)
    np.testing.assert_allclose(dnext - mu, lam, rtol=1e-15)


@pytest.mark.parametrize("k", [5, 40, 200])
def test_residual_bound(k):
    d, z, rho = random_system(np.random.default_rng(100 + k), k)
    sys, sol = _solve(d, z, rho)
    gam, mu = _np(sol.gamma), _np(sol.mu)
    G = _np(gap_table(np.arange(k), np.arange(k), d, sol.gamma, sol.mu))
    f = 1.0 + rho * (z[:, None] ** 2 / G).sum(0)
    bound = 64 * k * EPS * rho * np.sum(z ** 2) / np.minimum(gam, np.where(mu > 0, mu, np.inf))
    assert np.all(np.abs(f) <= bound)


@pytest.mark.parametrize("rho", [1.0, 3.7])
def test_weights_single_pole_any_rho(rho):
    sys, sol = _solve(np.array([0.2]), np.array([-0.6]), rho)
    zh = _np(hb.recompute_weights(sys.d, sol, sys.z, rho=rho))
    assert abs(zh[0] + 0.6) <= 1e-15 * 0.6


def test_weights_two_pole_hand_case():
    d, z, rho = _golden()
    sys, sol = _solve(d, z, rho)
    zh = _np(hb.recompute_weights(sys.d, sol, sys.z, rho=rho))
    lam = _np(sol.lam)
    u0 = np.sqrt((lam[1] - d[0]) / (d[1] - d[0]) * (lam[0] - d[0]))
    u1 = np.sqrt((lam[0] - d[1]) / (d[0] - d[1]) * (lam[1] - d[1]))
    np.testing.assert_allclose(np.abs(zh), [u0, u1], rtol=1e-14)
    np.testing.assert_allclose(np.abs(zh), np.abs(z), rtol=1e-13)


def test_weights_sign_convention():
    d, z, rho = random_system(np.random.default_rng(9), 9)
    sys, sol = _solve(d, z, rho)
    zh = _np(hb.recompute_weights(sys.d, sol, sys.z, rho=rho))
    np.testing.assert_array_equal(np.sign(zh), np.sign(z))


def test_stable_gap_branch_identities():
    d, z, rho = random_system(np.random.default_rng(15), 15)
    sys, sol = _solve(d, z, rho)
    gam, mu = _np(sol.gamma), _np(sol.mu)
    for i in range(15):
        assert stable_gap(i, i, d, gam, mu) == -gam[i]
        if i < 14:
            assert stable_gap(i + 1, i, d, gam, mu) == mu[i]
    G = _np(gap_table(np.arange(15), np.arange(15), d, sol.gamma, sol.mu))
    dext = np.append(d, d[-1] + gam[-1] + mu[-1])
    for i in range(15):
        for j in range(15):
            ref = (d[i] - d[j]) - gam[j] if i <= j else (d[i] - dext[j + 1]) + mu[j]
            assert G[i, j] == ref


def test_stable_gap_matches_naive_when_separated():
    d, z, rho = random_system(np.random.default_rng(12), 12, span=12.0)
    sys, sol = _solve(d, z, rho)
    G = _np(gap_table(np.arange(12), np.arange(12), d, sol.gamma, sol.mu))
    naive = d[:, None] - _np(sol.lam)[None, :]
    assert np.all(np.abs(G - naive) <= 1e-8 * np.abs(naive))


def test_eigvec_golden_and_single_pole():
    for d, z, rho in (_golden(), (np.array([0.5]), np.array([2.0]), 1.0)):
        sys, sol = _solve(d, z, rho)
        hb.recompute_weights(sys.d, sol, sys.z, rho=rho)
        C = hb.CauchyEvecMatrix.from_secular(sys, sol)
        Q = _np(C.to_dense())
        assert np.abs(Q.T @ Q - np.eye(d.size)).max() <= 1e-15
        assert np.all(np.isfinite(_np(sol.v)))
