"""Edge cases of the full solver (mirrors pkg/tests/test_dc.py: n = 1, exact decoupling,
small closed forms, the HSS path on Toeplitz 2000, Clement metrics, path equivalence,
threshold degeneration, record / flop diagnostics) on the level-batched GPU solver."""
import numpy as np
import pytest
import torch

import paper_1510_04591_b200 as hb

pytestmark = pytest.mark.gpu


def _dense(T):
    n = T.n
    A = np.diag(T.a)
    if n > 1:
        A += np.diag(T.b, 1) + np.diag(T.b, -1)
    return A


def test_solve_n1():
    res = hb.adc_solve(hb.SymTridiagonal(np.array([-2.5]), np.zeros(0)))
    assert res.lam[0] == -2.5 and float(res.Q[0, 0]) == 1.0


def test_solve_rejects_nonfinite():
    with pytest.raises(ValueError):
        hb.adc_solve(hb.SymTridiagonal(np.array([np.nan, 1.0]), np.array([1.0])))


def test_decoupled_solver_returns_union():
    # test_dc.py:85-91: an exactly zero coupling splits the problem
    a = np.array([3.0, 1.0, 4.0, 1.5, 9.0, 2.6])
    b = np.array([0.4, 0.3, 0.0, 0.2, 0.1])
    T = hb.SymTridiagonal(a, b)
    res = hb.adc_solve(T, hb.SolverConfig(base_size=3, method="dense-dc"))
    ref = np.linalg.eigvalsh(_dense(T))
    assert np.abs(res.lam - ref).max() <= 1e-13 * T.norm_max()
    Q = res.Q.cpu().numpy()
    assert np.abs(_dense(T) @ Q - Q * res.lam).max() <= 1e-13 * T.norm_max()


def test_toeplitz_n8_closed_form():
    res = hb.adc_solve(hb.gen_toeplitz(8), hb.SolverConfig(base_size=3, method="dense-dc"))
    closed = np.sort(2.0 + 2.0 * np.cos(np.arange(1, 9) * np.pi / 9.0))
    assert np.abs(res.lam - closed).max() <= 1e-14


def test_solve_toeplitz_2000_hss_path():
    # test_dc.py:249-257
    T = hb.gen_toeplitz(2000)
    cfg = hb.SolverConfig(method="adc-rand", hss_threshold=400, leaf_size=100, seed=3)
    res = hb.adc_solve(T, cfg)
    closed = np.sort(2.0 + 2.0 * np.cos(np.arange(1, 2001) * np.pi / 2001.0))
    assert np.abs(res.lam - closed).max() <= 1e-12
    assert any(m.used_hss for m in res.merges)
    assert np.all(np.diff(res.lam) >= 0)
    assert float((torch.linalg.norm(res.Q, dim=0) - 1.0).abs().max()) <= 1e-13


def test_solve_clement_1500_metrics():
    # test_dc.py:260-268
    T = hb.gen_clement(1500)
    cfg = hb.SolverConfig(method="adc-rand", hss_threshold=400, leaf_size=100, seed=0)
    res = hb.adc_solve(T, cfg)
    n = 1500
    Q = res.Q
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    assert float((Q.T @ Q - I).abs().max()) / n <= 1e-11
    A = torch.as_tensor(_dense(T), device="cuda")
    lam = torch.as_tensor(res.lam, device="cuda")
    back = float((A - (Q * lam) @ Q.T).abs().max()) / (T.norm_max() * n)
    assert back <= 1e-12


def test_path_equivalence():
    # test_dc.py:271-277
    rng = np.random.default_rng(11)
    T = hb.SymTridiagonal(rng.uniform(-1, 1, 700), rng.uniform(-1, 1, 699))
    kw = dict(hss_threshold=400, leaf_size=100, seed=5)
    lam_d = hb.adc_solve(T, hb.SolverConfig(method="dense-dc", **kw)).lam
    lam_a = hb.adc_solve(T, hb.SolverConfig(method="adc-rand", **kw)).lam
    assert np.abs(lam_d - lam_a).max() <= 1e-12 * T.norm_max()


def test_threshold_above_n_degenerates_to_dense():
    # test_dc.py:280-288: no merge reaches the threshold -> identical results and counts
    rng = np.random.default_rng(12)
    T = hb.SymTridiagonal(rng.uniform(-1, 1, 300), rng.uniform(-1, 1, 299))
    res_d = hb.adc_solve(T, hb.SolverConfig(method="dense-dc", seed=9))
    res_a = hb.adc_solve(T, hb.SolverConfig(method="adc-rand", hss_threshold=2000, seed=9))
    np.testing.assert_array_equal(res_d.lam, res_a.lam)
    assert torch.equal(res_d.Q, res_a.Q)
    assert res_d.flops.as_dict() == res_a.flops.as_dict()


def test_diagnostics_populated():
    # test_dc.py:291-296
    rng = np.random.default_rng(13)
    T = hb.SymTridiagonal(rng.uniform(-1, 1, 200), rng.uniform(-1, 1, 199))
    res = hb.adc_solve(T, hb.SolverConfig(method="dense-dc"))
    assert res.merges and all(m.size >= 2 for m in res.merges)
    assert 0.0 <= res.max_deflation_fraction() <= 1.0
    assert res.flops.secular > 0 and res.flops.update_dense > 0


@pytest.mark.parametrize("n", [2, 3, 26, 27, 51, 777])
def test_ragged_sizes_match_lapack(n):
    # uneven splits, leaves of different depths, and the smallest merges
    rng = np.random.default_rng(n)
    T = hb.SymTridiagonal(rng.uniform(-1, 1, n), rng.uniform(0.1, 1, n - 1))
    res = hb.adc_solve(T, hb.SolverConfig(base_size=3 if n < 30 else 25))
    ref = np.linalg.eigvalsh(_dense(T))
    assert np.abs(res.lam - ref).max() <= 1e-13 * T.norm_max() * max(1, np.log2(n))
    Q = res.Q.cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-13 * n


def test_level_batched_hss_equals_one_merge_at_a_time():
    # the level's HSS merges run phase by phase on side streams (dc.update_vectors_hss_many);
    # every output must be bit-identical to update_vectors_hss called merge by merge
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import config4_system
    from paper_1510_04591_b200 import secular
    from paper_1510_04591_b200.cauchy import CauchyEvecMatrix
    from paper_1510_04591_b200.dc import HssJob, MergeRecord, update_vectors_hss, update_vectors_hss_many
    from paper_1510_04591_b200.flops import FlopCounter
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
    jobs, refs = [], []
    for i, n in enumerate([700, 1024, 1500, 900, 2048, 640, 1200, 800, 1300]):
        d, u, rho = config4_system(n, 20 + i)
        s = secular.RankOneSystem(d, u, rho)
        sol = secular.solve_secular(s)
        secular.recompute_weights(s.d, sol, s.z, rho=rho)
        C = CauchyEvecMatrix.from_secular(s, sol)
        Q = torch.as_tensor(np.random.default_rng(i).standard_normal((n + 17, n)), device="cuda")
        rec1, rec2 = MergeRecord(size=n, kept=n, n_deflated=0), MergeRecord(size=n, kept=n, n_deflated=0)
        f1, f2 = FlopCounter(), FlopCounter()
        refs.append((update_vectors_hss(Q, C, cfg, seed=[3, i], flops=f1, record=rec1), rec1, f1))
        jobs.append(HssJob(Q=Q, C=C, seed=[3, i], flops=f2, record=rec2, d=C.d.cpu().numpy(),
                           gamma=C.gamma.cpu().numpy(), mu=C.mu.cpu().numpy(),
                           out=torch.empty(n + 17, n, dtype=torch.float64, device="cuda")))
    update_vectors_hss_many(jobs, cfg, max_streams=4)
    torch.cuda.synchronize()
    assert any(r.used_hss for _, r, _ in refs)
    for (ref, rec1, f1), j in zip(refs, jobs):
        assert torch.equal(ref, j.out)
        assert (rec1.used_hss, rec1.fell_back, rec1.hss_rank) == \
            (j.record.used_hss, j.record.fell_back, j.record.hss_rank)
        assert f1.as_dict() == j.flops.as_dict()
