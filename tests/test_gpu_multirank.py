"""Two ranks on the one GPU of this box (gloo for the host-side collectives): the
multi-GPU drivers with the real device ops (GpuOps: every kernel through the C ABI)
against the single-process GPU results.  The ranks never wait on each other inside a
kernel; NCCL's own path is exercised by the one-rank tests in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path, peer="1"):
    os.environ["HSSEIG_PEER"] = peer
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200.distributed import GpuOps, ShardedMerge, adc_solve_distributed
    from helpers import config4_system
    n = 2048
    d, u, rho = config4_system(n, 5)
    X = torch.as_tensor(np.random.default_rng(3).standard_normal((64, n)), device="cuda")
    r0, r1 = rank * 64 // world, (rank + 1) * 64 // world
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
    sm = ShardedMerge(n, cfg, GpuOps(n))
    lam, out, info = sm.run(torch.as_tensor(d, device="cuda"), torch.as_tensor(u, device="cuda"),
                            rho, X[r0:r1].contiguous(), seed=[0, 7])
    cfg1 = hb.SolverConfig(leaf_size=64, hss_threshold=256, method="adc-srrsc")
    ops1 = GpuOps(n)
    _, out1, info1 = ShardedMerge(n, cfg1, ops1).run(
        torch.as_tensor(d, device="cuda"), torch.as_tensor(u, device="cuda"), rho,
        X[r0:r1].contiguous(), seed=[0, 7])
    T = hb.gen_config5(1024, 4)
    ops5 = GpuOps(512)
    res = adc_solve_distributed(T, hb.SolverConfig(rank_eps=1e-13), ops5)
    # the sample rows went straight into both ranks' Y / Z (CUDA IPC peer stores fused in
    # the split-K reduction), not through a separate all-gather
    assert info.get("sample_gather") == ("peer" if peer == "1" else "nccl"), info.get("sample_gather")
    outs = [None] * world
    dist.all_gather_object(outs, (out.cpu().numpy(), res.row0, res.row1, res.Q_rows.cpu().numpy(),
                                  out1.cpu().numpy(), bool(info1["used_hss"])))
    if rank == 0:
        Q = np.zeros((1024, 1024))
        for _, a, b, q, _, _ in outs:
            Q[a:b] = q
        np.savez(out_path, lam=lam.cpu().numpy(), out=np.concatenate([o[0] for o in outs]),
                 used=info["used_hss"], elam=res.lam, Q=Q,
                 out1=np.concatenate([o[4] for o in outs]), used1=all(o[5] for o in outs))
    # the CUDA-IPC peer buffers are unmapped in group order before the processes exit
    for ops in (sm.ops, ops1, ops5):
        ops.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("peer", ["1", "0"])
def test_two_ranks_match_single_gpu(tmp_path, peer):
    # peer = "1": sample rows stored into both ranks' Y / Z by the reduction kernels (CUDA
    # IPC); "0": the NCCL-style all-gather fallback (gloo here)
    import paper_1510_04591_b200 as hb
    from helpers import config4_system
    out_path = str(tmp_path / "mr.npz")
    mp.spawn(_worker, args=(2, _port(), out_path, peer), nprocs=2, join=True)
    r = np.load(out_path)
    n = 2048
    d, u, rho = config4_system(n, 5)
    X = torch.as_tensor(np.random.default_rng(3).standard_normal((64, n)), device="cuda")
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
    lam, ref, _ = hb.merge_update(d, u, rho, X, cfg, seed=[0, 7])
    assert bool(r["used"])
    np.testing.assert_allclose(r["lam"], lam.cpu().numpy(), rtol=0, atol=64 * 2.2e-16 * np.abs(r["lam"]).max())
    refn = ref.cpu().numpy()
    np.testing.assert_allclose(r["out"], refn, rtol=0, atol=1e-12 * np.abs(refn).max())
    # ADC1 (SRRSC construction partitioned by subtree, slots all-gathered)
    cfg1 = hb.SolverConfig(leaf_size=64, hss_threshold=256, method="adc-srrsc")
    _, ref1, _ = hb.merge_update(d, u, rho, X, cfg1, seed=[0, 7])
    assert bool(r["used1"])
    ref1 = ref1.cpu().numpy()
    np.testing.assert_allclose(r["out1"], ref1, rtol=0, atol=1e-12 * np.abs(ref1).max())
    T = hb.gen_config5(1024, 4)
    res = hb.adc_solve(T, hb.SolverConfig(rank_eps=1e-13))
    np.testing.assert_allclose(r["elam"], res.lam, rtol=0, atol=1e-13 * T.norm_max())
    Qs = res.Q.cpu().numpy()
    sg = np.sign((r["Q"] * Qs).sum(0))
    np.testing.assert_allclose(r["Q"] * sg, Qs, rtol=0, atol=1e-12)
