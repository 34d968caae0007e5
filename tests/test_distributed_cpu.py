"""World-size-2 gloo test of the multi-GPU merge driver's host logic (sharding, padding,
all-gathers, replicated construction, row-local multiply) with a NumPy stand-in for the
device ops (the oracle).  The GPU path runs the same driver with GpuOps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import config4_system
from oracle import hss_oracle as orc


class NumpyOps:
    """Oracle-backed ops: each 'part' is the full oracle result sliced to the shard."""
    max_width = 112

    def __init__(self, k):
        self.k = k

    def secular_part(self, d, z, rho, lo, hi):
        lam, gam, mu, _, per = orc.secular_all(d.numpy(), z.numpy(), rho, per_root=True)
        sl = slice(lo, hi)
        bad_g = lo + int(np.flatnonzero(gam[sl] <= 0)[0]) if np.any(gam[sl] <= 0) else self.k
        bad_m = lo + int(np.flatnonzero(mu[sl] <= 0)[0]) if np.any(mu[sl] <= 0) else self.k
        st = torch.tensor([int(per[sl].sum()), bad_g, bad_m], dtype=torch.int64)
        return (torch.as_tensor(lam[sl]), torch.as_tensor(gam[sl]), torch.as_tensor(mu[sl]), st)

    def dnext(self, d, gam, mu):
        return torch.cat([d[1:], (d[-1:] + gam[-1:]) + mu[-1:]])

    def loewner_part(self, d, dn, gam, mu, z, rho, lo, hi):
        zh = orc.loewner(d.numpy(), gam.numpy(), mu.numpy(), z.numpy(), rho)
        return torch.as_tensor(zh[lo:hi]), torch.tensor([self.k], dtype=torch.int64)

    def normalizers_part(self, d, dn, gam, mu, zh, lo, hi):
        v = orc.normalizers(d.numpy(), gam.numpy(), mu.numpy(), zh.numpy())
        return torch.as_tensor(v[lo:hi])

    def generators(self, d, dn, gam, mu, zh, v):
        return orc.Generators(d.numpy(), gam.numpy(), mu.numpy(), zh.numpy(), v.numpy())

    def omega(self, seed, k, w):
        return torch.as_tensor(orc.sample_block(k, w, seed))

    def _yz(self, G, om, part):
        if part is not None:           # the off-diagonal sample
            return orc.offdiag_samples(G, list(part.ranges), om.numpy())
        return G.times(om.numpy()), G.t_times(om.numpy())

    def sample_part(self, G, om, w, lo, hi, part=None):
        Y, Z = self._yz(G, om, part)
        return torch.as_tensor(Y[lo:hi]), torch.as_tensor(Z[lo:hi])

    def build(self, G, part, w, om, Y, Z, group=None, offdiag=True):
        # the gathered samples must be the full (off-diagonal) products
        Yr, Zr = self._yz(G, om, part if offdiag else None)
        assert np.allclose(Y.numpy(), Yr, rtol=0, atol=1e-13)
        assert np.allclose(Z.numpy(), Zr, rtol=0, atol=1e-13)
        return orc.rand_construct(G, list(part.ranges), w - 10, 10, Omega=om.numpy(),
                                  offdiag=offdiag)

    def build_srrsc(self, G, part, cap, tol, group=None):
        from oracle import srrsc_oracle as so
        return so.srrsc_construct(G, list(part.ranges), cap, tol)

    def flagged(self, T):
        return T.flagged

    def r_used(self, T):
        return T.r_used

    def construct_flops(self, T):
        return 0

    def mult_flops(self, T, P):
        return 0

    def multiply(self, X, T):
        return torch.as_tensor(orc.hss_apply_right(X.numpy(), T))

    def dense(self, X, G):
        return torch.as_tensor(orc.update_dense(X.numpy(), G))


def _worker(rank, world, port, k, P, out_path, method="adc-rand"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_04591_b200 import SolverConfig
    from paper_1510_04591_b200.distributed import ShardedMerge
    d, u, rho = config4_system(k, 3)
    X = np.random.default_rng(7).standard_normal((P, k))
    r0, r1 = rank * P // world, (rank + 1) * P // world
    cfg = SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13, method=method)
    sm = ShardedMerge(k, cfg, NumpyOps(k))
    lam, out, info = sm.run(torch.as_tensor(d), torch.as_tensor(u), rho, torch.as_tensor(X[r0:r1]),
                            seed=[0, 0])
    parts = [torch.empty(((r + 1) * P // world - r * P // world, k), dtype=torch.float64)
             for r in range(world)]
    if out.shape[0] < parts[rank].shape[0]:
        raise AssertionError("bad local shape")
    dist.all_gather(parts, out.contiguous()) if len({p.shape for p in parts}) == 1 else None
    if rank == 0:
        np.savez(out_path, lam=lam.numpy(), out=torch.cat(parts).numpy(),
                 used=info["used_hss"], r=info["r_used"])
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("k,P", [(600, 40)])
def test_sharded_merge_world2_matches_single_process(tmp_path, k, P):
    out_path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), k, P, out_path), nprocs=2, join=True)
    res = np.load(out_path)
    d, u, rho = config4_system(k, 3)
    X = np.random.default_rng(7).standard_normal((P, k))
    G, lam, _ = orc.generators_from_roots(d, u, rho)
    ref = orc.update_hss(X, G, 64, 10, 1e-13, 100, [0, 0], offdiag=True)
    assert bool(res["used"])
    np.testing.assert_array_equal(res["lam"], lam)
    np.testing.assert_allclose(res["out"], ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_sharded_merge_adc1_world2_matches_single_process(tmp_path):
    # ADC1 through the same sharded driver: gathered generators, SRRSC tree, row-local product
    from oracle import srrsc_oracle as so
    k, P = 600, 40
    out_path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), k, P, out_path, "adc-srrsc"), nprocs=2, join=True)
    res = np.load(out_path)
    d, u, rho = config4_system(k, 3)
    X = np.random.default_rng(7).standard_normal((P, k))
    G, lam, _ = orc.generators_from_roots(d, u, rho)
    ref = so.update_srrsc(X, G, 64, 1e-15)
    assert bool(res["used"])
    np.testing.assert_array_equal(res["lam"], lam)
    np.testing.assert_allclose(res["out"], ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_shard_ranges_cover_exactly():
    from paper_1510_04591_b200.distributed import shard_range
    for k in (1, 7, 600, 32768):
        for world in (1, 2, 3, 8):
            got = [shard_range(k, r, world)[:2] for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))


def test_subtree_layout_matches_postorder():
    from paper_1510_04591_b200.distributed import subtree_layout
    from oracle.hss_oracle import postorder_nodes
    for depth in (1, 2, 3, 5):
        ranges = [(i, i + 1) for i in range(1 << depth)]
        nodes, root = postorder_nodes(ranges)
        for s_lev in range(0, depth + 1):
            blocks, leaves = subtree_layout(depth, s_lev)
            assert len(blocks) == 1 << s_lev
            for (a, b), (la, lb) in zip(blocks, leaves):
                sub = nodes[b - 1]          # subtree root is last in its postorder block
                assert sub.level == s_lev
                assert all(sub.lo <= nodes[i].lo and nodes[i].hi <= sub.hi for i in range(a, b))
                assert (sub.lo, sub.hi) == (la, lb)


class NumpySolveOps(NumpyOps):
    """NumpyOps plus the full-solve pieces: oracle subtree solves, NumPy row-block glue;
    the host deflation is the library's own C function (hsseig_wave_deflate)."""
    device = "cpu"

    def __init__(self):
        super().__init__(0)

    def tensor(self, x):
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64))

    def secular_part(self, d, z, rho, lo, hi):
        self.k = d.numel()
        return super().secular_part(d, z, rho, lo, hi)

    def local_solve(self, a, b, nodes, sub, cfg):
        from paper_1510_04591_b200.distributed import _split_a
        nd = nodes[sub]
        a_top = _split_a(a, b, nodes, nd["depth"])
        lo, hi = nd["lo"], nd["hi"]
        lam, Q, _, _ = orc.adc_solve(a_top[lo:hi], b[lo:hi - 1], orc.Config(base_size=cfg.base_size))
        return lam, torch.as_tensor(Q), {}

    def deflate(self, nL, nR, L, zrow, bk):
        from paper_1510_04591_b200 import _native as nat
        from paper_1510_04591_b200.distributed import deflate_merge
        return deflate_merge(nat.load(build_if_missing=False), nL, nR, L, zrow, bk)

    def assemble_rows(self, Qc, coff, nc, src, n):
        Q = Qc.numpy()
        sc = src - coff
        ok = (sc >= 0) & (sc < nc)
        W = np.zeros((Q.shape[0], n))
        W[:, ok] = Q[:, sc[ok]]
        return torch.as_tensor(W)

    def rotate(self, W, ca, cb, c, s):
        w = W.numpy()
        for i, j, cc, ss in zip(ca, cb, c, s):
            x, y = w[:, i].copy(), w[:, j].copy()
            w[:, i] = cc * x + ss * y
            w[:, j] = -ss * x + cc * y

    def gather(self, Qk, W, order, k):
        w = W.numpy()
        out = np.empty_like(w)
        for c, sc in enumerate(order):
            out[:, c] = Qk.numpy()[:, sc] if sc < k else w[:, sc]
        return torch.as_tensor(out)


def _solve_worker(rank, world, port, n, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_04591_b200 import SolverConfig
    from paper_1510_04591_b200.distributed import adc_solve_distributed
    from paper_1510_04591_b200.matgen import gen_config5
    T = gen_config5(n, 1)
    res = adc_solve_distributed(T, SolverConfig(), NumpySolveOps())
    rows = [torch.empty(0) for _ in range(world)]
    dist.all_gather_object(rows, (res.row0, res.row1, res.Q_rows.numpy()))
    if rank == 0:
        Q = np.zeros((n, n))
        for r0, r1, q in rows:
            Q[r0:r1] = q
        np.savez(out_path, lam=res.lam, Q=Q, nmerges=len(res.merges))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 200), (4, 430)])
def test_distributed_full_solve_matches_oracle(tmp_path, world, n):
    # multi-GPU config-5 solve logic: subtrees per rank, row-block sharded top merges
    from paper_1510_04591_b200.matgen import gen_config5
    out_path = str(tmp_path / "solve.npz")
    mp.spawn(_solve_worker, args=(world, _free_port(), n, out_path), nprocs=world, join=True)
    res = np.load(out_path)
    T = gen_config5(n, 1)
    lam, Q, infos, _ = orc.adc_solve(T.a, T.b, orc.Config())
    assert int(res["nmerges"]) == world - 1      # the shared top merges (subtree records are the oracle's)
    np.testing.assert_allclose(res["lam"], lam, rtol=0, atol=1e-13)
    Qd = res["Q"]
    s = np.sign((Qd * Q).sum(0))
    np.testing.assert_allclose(Qd * s, Q, rtol=0, atol=1e-12)


def _bench_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rec = bench.eigh_distributed(world, ops=NumpySolveOps(), device="cpu", n=240, warm=False)
    if rank == 0:
        np.savez(out_path, **{k: np.asarray(v) for k, v in rec.items()})
    dist.destroy_process_group()


def test_bench_distributed_eigh_line_world2(tmp_path):
    # the bench's config-5 multi-GPU line (halo residual, sampled orthogonality, max-over-ranks
    # wall time) with gloo and the oracle stand-in
    out_path = str(tmp_path / "b.npz")
    mp.spawn(_bench_worker, args=(2, _free_port(), out_path), nprocs=2, join=True)
    r = np.load(out_path)
    assert int(r["ranks"]) == 2 and float(r["wall_s"]) > 0
    assert float(r["orthogonality"]) < 1e-15 and float(r["residual"]) < 1e-15
