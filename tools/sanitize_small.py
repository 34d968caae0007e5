"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs every kernel family once at sizes the sanitizer finishes in minutes: secular /
Loewner / normalizers, the device Gaussian draw, the Cauchy panel + TMA/DMMA sampling
GEMMs (split-K reductions), the ID and level-batched construction (both sample modes),
the HSS multiply (narrow and wide TMA ring tiles), the fused dense update, ADC1 (SRRSC
clusters), the batched base-case QL and the level-batched solver glue (assemble /
rotate / gather), and the one-rank sharded merge.
    compute-sanitizer --tool memcheck python tools/sanitize_small.py [part]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1510_04591_b200 as hb  # noqa: E402
from paper_1510_04591_b200 import hss  # noqa: E402
from paper_1510_04591_b200.matgen import isolated_merge_system  # noqa: E402

part = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)


def merge(k, leaf, sample, method="adc-rand"):
    d, u, rho = isolated_merge_system(k, 3)
    X = torch.as_tensor(np.random.default_rng(1).standard_normal((200, k)), device="cuda")
    cfg = hb.SolverConfig(leaf_size=leaf, hss_threshold=4 * leaf, rank_eps=1e-13, sample=sample,
                          method=method)
    rec = hb.MergeRecord(size=k, kept=k, n_deflated=0)
    lam, Qn, _ = hb.merge_update(d, u, rho, X, cfg, seed=[0, 1], record=rec)
    torch.cuda.synchronize()
    print(f"merge k={k} leaf={leaf} {method}/{sample}: used_hss={rec.used_hss} "
          f"rank={rec.hss_rank} fell_back={rec.fell_back}", flush=True)


if part in ("all", "merge"):
    merge(1024, 128, "offdiag")
    merge(1024, 64, "reference")
    merge(700, 64, "offdiag")                        # ragged leaves, odd starts
    merge(1024, 128, "offdiag", method="adc-srrsc")
    merge(600, 64, "offdiag", method="dense-dc")

if part in ("all", "mult"):
    d, u, rho = isolated_merge_system(2048, 4)
    s = hb.RankOneSystem(d, u, rho)
    sol = hb.solve_secular(s)
    hb.recompute_weights(d, sol, u, rho=rho)
    C = hb.CauchyEvecMatrix.from_secular(s, sol)
    p = hb.build_partition(2048, 128, C.d, C.gamma, C.mu)
    r = min(hb.estimate_rank(p, C.d, C.gamma, C.mu, 1e-13, 100), p.min_leaf - 10)
    H = hb.rand_hss_construct(C, p, r, p=10, seed=[0, 0])
    X = torch.randn(300, 2048, dtype=torch.float64, device="cuda")
    Y = hss.hss_matmul_right(X, H)
    Yd = hb.update_vectors_dense(X, C.to_dense())
    torch.cuda.synchronize()
    print("mult err", float((Y - Yd).abs().max()), flush=True)

if part in ("all", "solve"):
    for T in (hb.gen_toeplitz(600), hb.gen_kac(512), hb.gen_uniform(700, 2)):
        for m in ("adc-rand", "dense-dc", "adc-srrsc"):
            res = hb.adc_solve(T, hb.SolverConfig(method=m, leaf_size=64, hss_threshold=256,
                                                  rank_eps=1e-13))
            torch.cuda.synchronize()
            print(f"solve n={T.n} {m}: merges {len(res.merges)} "
                  f"hss {sum(x.used_hss for x in res.merges)}", flush=True)

if part in ("all", "shard"):
    import torch.distributed as dist
    from paper_1510_04591_b200.distributed import GpuOps, ShardedMerge
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    d, u, rho = isolated_merge_system(1024, 5)
    X = torch.as_tensor(np.random.default_rng(3).standard_normal((64, 1024)), device="cuda")
    sm = ShardedMerge(1024, hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13),
                      GpuOps(1024))
    lam, out, info = sm.run(torch.as_tensor(d, device="cuda"), torch.as_tensor(u, device="cuda"),
                            rho, X, seed=[0, 7])
    torch.cuda.synchronize()
    print("sharded merge used_hss", info["used_hss"], flush=True)
    dist.destroy_process_group()
print("sanitize driver done", flush=True)
