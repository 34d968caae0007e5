"""BASELINE.json's configurations at their full sizes, through size-independent properties
(the CPU oracle cannot finish them in test time): closed-form spectra, trace, orthogonality
and eigen-residuals, root interlacing, and the HSS update against the dense update of the
same merge."""
import numpy as np
import pytest
import torch

import paper_1510_04591_b200 as hb

from helpers import config4_system

pytestmark = pytest.mark.gpu


def _orth_sampled(Q, cols, seed=0):
    """max |Q_S^T Q_S - I| / n over a seeded column sample S (exact when S is everything)."""
    n = Q.shape[1]
    if cols >= n:
        S = torch.arange(n, device=Q.device)
    else:
        S = torch.as_tensor(np.sort(np.random.default_rng(seed).choice(n, cols, replace=False)),
                            device=Q.device)
    Qs = Q[:, S]
    G = Qs.T @ Qs
    G.diagonal().sub_(1.0)
    return float(G.abs().max()) / n


def _residual(T, lam, Q):
    """max |T Q - Q diag(lam)| / (n max|T|) (BASELINE's residual, entrywise-max convention)."""
    a = torch.as_tensor(T.a, device="cuda")
    b = torch.as_tensor(T.b, device="cuda")
    TQ = a[:, None] * Q
    TQ[:-1] += b[:, None] * Q[1:]
    TQ[1:] += b[:, None] * Q[:-1]
    TQ -= Q * torch.as_tensor(lam, device="cuda")[None, :]
    return float(TQ.abs().max()) / (T.n * T.norm_max())


def test_config4_merge_full_size_matches_dense_update():
    # BASELINE config 4: N = 32768, leaf 128, tol 1e-13; Q_old = QR of a Gaussian
    n = 32768
    d, u, rho = config4_system(n, 0)
    g = torch.Generator(device="cuda").manual_seed(0)
    Q0, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    cfg = hb.SolverConfig(leaf_size=128, hss_threshold=512, rank_eps=1e-13)
    rec = hb.MergeRecord(size=n, kept=n, n_deflated=0)
    lam, Qn, C = hb.merge_update(d, u, rho, Q0, cfg, seed=[0, 0], record=rec)
    assert rec.used_hss and not rec.fell_back and rec.hss_rank <= 112
    # interlacing of the roots with the poles (rho > 0)
    lam_h = lam.cpu().numpy()
    assert np.all(lam_h > d) and np.all(lam_h[:-1] < d[1:])
    # the structured product against the dense product with the same generators
    Qd = hb.update_vectors_dense(Q0, C)
    assert float((Qn - Qd).abs().max()) <= 1e-12
    del Qd
    assert _orth_sampled(Qn, 4096) <= 1e-15
    # eigen-residual of diag(d) + rho u u^T on a row sample of Q0^T Qn
    M = Q0.T @ Qn                      # = the HSS approximation of C
    dd = torch.as_tensor(d, device="cuda")
    uu = torch.as_tensor(u, device="cuda")
    uM = uu @ M
    rows = torch.as_tensor(np.random.default_rng(1).choice(n, 512, replace=False), device="cuda")
    R = dd[rows, None] * M[rows] + rho * uu[rows, None] * uM[None, :] - M[rows] * lam[None, :]
    assert float(R.abs().max()) <= 1e-11


@pytest.mark.parametrize("method", ["adc-srrsc", "adc-rand"])
def test_config2_toeplitz_full_size(method):
    # BASELINE config 2 (ADC1 as named, and ADC2): 2 + 2 cos(j pi / (N+1))
    n = 10000
    T = hb.gen_toeplitz(n)
    res = hb.adc_solve(T, hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13,
                                          method=method))
    ref = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.abs(res.lam - ref).max() <= 1e-12 * T.norm_max()
    assert sum(m.used_hss for m in res.merges) > 0
    if method == "adc-srrsc":
        assert res.merges[-1].used_hss     # ADC1 compresses the k = 5000 top merge
    assert _orth_sampled(res.Q, n) <= 1e-15
    assert _residual(T, res.lam, res.Q) <= 1e-15


def test_config3_kac_full_size():
    # BASELINE config 3 (Clement/Kac form): eigenvalues -(N-1) + 2j
    n = 20000
    T = hb.gen_kac(n)
    res = hb.adc_solve(T, hb.SolverConfig(rank_eps=1e-13))
    ref = -(n - 1) + 2.0 * np.arange(n)
    assert np.abs(res.lam - ref).max() <= 1e-12 * T.norm_max()
    assert res.merges[-1].used_hss
    assert _orth_sampled(res.Q, 8192) <= 1e-15
    assert _residual(T, res.lam, res.Q) <= 1e-15


def test_config5_full_size():
    # BASELINE config 5 on one GPU: N = 65536, d ~ U(0,1), e ~ U(0.5,1)
    n = 65536
    T = hb.gen_config5(n, 0)
    res = hb.adc_solve(T, hb.SolverConfig(rank_eps=1e-13))
    lam = res.lam
    assert np.all(np.diff(lam) >= 0)
    # Gershgorin / trace checks that need no reference
    assert abs(lam.sum() - T.a.sum()) <= 1e-10 * n
    assert _residual(T, lam, res.Q) <= 1e-15
    assert _orth_sampled(res.Q, 4096) <= 1e-15
