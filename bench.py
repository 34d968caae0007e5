"""Benchmark: BASELINE config 4 — isolated top-level DC merge, N = 32768, on B200.

One step = one pass of the merge hot path (secular roots -> Loewner weights ->
column normalizers -> partition / rank estimate -> Omega -> off-diagonal sample
-> randomized HSS construction -> Q_new = Q_old H) over one synthetic input.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value  = FP64 TF/s of the merge with inputs resident in HBM, counted as the REFERENCE's
         work for this exact input: its FlopCounter (pkg/src/hsseig/flops.py) over its own
         tree, recorded by tests/golden/make_golden_configs.py (c4_32768), divided by our
         wall time.  Our tree is smaller (the off-diagonal sample), so the
         flops we execute are reported beside it ("flops", "value_own_tree"); the roofline
         uses the executed flops of the multiply kernel.
e2e    = the same through the public API with Q_old / d / u in pinned host memory,
         H2D and D2H copies inside the timed region.
N > 1 (torchrun): the rows of Q_old are sharded across ranks (row-block sharding);
the merge factors are computed per rank and the multiply is row-local.
--impl reference: the reference itself (baseline/_ref, built from /root/reference/pkg by
its own setup; the oracle port when absent) on the host cores, on a bounded sample of the
workload: the config-4 merge at N = 4096, stamped as such in its config.
"""
import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_MERGE = 32768
LEAF = 128
RANK_EPS = 1e-13
OVERSAMPLE = 10
SEED = 0
CPU_SAMPLE_N = 4096
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # HSSEIG_BENCH_N: the same under torchrun (whose parser takes --n for its own options)
    ap.add_argument("--n", type=int, default=int(os.environ.get("HSSEIG_BENCH_N", N_MERGE)))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-eigh", action="store_true")
    ap.add_argument("--cpu-eigh-all", action="store_true",
                    help="also time the reference's config-3 solve on the host (~2 min)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- CPU arm
def reference_module():
    """The unmodified reference package (baseline/_ref), or None when it was not built."""
    if not os.path.isdir(os.path.join(REF_DIR, "hsseig")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import hsseig
        import hsseig.dc  # noqa: F401
        import hsseig.hss  # noqa: F401
    except ImportError:
        return None
    return hsseig


def cpu_merge(n):
    """One config-4-shaped merge on the host: the reference's own chain (secular ->
    Loewner -> normalizers -> partition / rank -> rand_hss_construct -> hss_matmul_right
    over all n rows of Q_old) when baseline/_ref exists, else the oracle port.  Returns
    (TF/s, seconds, reference flops, kind)."""
    from paper_1510_04591_b200.matgen import isolated_merge_system
    d, u, rho = isolated_merge_system(n, SEED)
    Q0 = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))[0]
    h = reference_module()
    if h is not None:
        from hsseig import hss
        from hsseig.cauchy import CauchyEvecMatrix
        from hsseig.flops import FlopCounter
        from hsseig.secular import RankOneSystem, recompute_weights, solve_secular
        f = FlopCounter()
        t0 = time.perf_counter()
        sys_ = RankOneSystem(d, u, rho)
        sol = solve_secular(sys_, flops=f)
        recompute_weights(sys_.d, sol, sys_.z, rho=rho, flops=f)
        C = CauchyEvecMatrix.from_secular(sys_, sol, flops=f)
        part = hss.build_partition(C.k, LEAF, C.d, C.gamma, C.mu)
        r = min(hss.estimate_rank(part, C.d, C.gamma, C.mu, RANK_EPS, 100), part.min_leaf - OVERSAMPLE)
        H = hss.rand_hss_construct(C, part, r, p=OVERSAMPLE, seed=[SEED, 0], flops=f)
        hss.hss_matmul_right(Q0, H, flops=f)
        dt = time.perf_counter() - t0
        fl = f.secular + f.hss_construct + f.hss_mult + f.update_dense
        return fl / dt / 1e12, dt, fl, "reference"
    from oracle import hss_oracle as orc
    f = orc.Flops()
    t0 = time.perf_counter()
    G, lam, _ = orc.generators_from_roots(d, u, rho, f)
    orc.update_hss(Q0, G, LEAF, OVERSAMPLE, RANK_EPS, 100, [SEED, 0], f)
    dt = time.perf_counter() - t0
    fl = f.secular + f.hss_construct + f.hss_mult + f.update_dense
    return fl / dt / 1e12, dt, fl, "port"


def cpu_eigh(names):
    """The reference's full adc_solve on BASELINE configs on the host (wall-s, the core
    count of this host); returns {} when baseline/_ref is absent."""
    h = reference_module()
    if h is None:
        return {}
    from hsseig.matgen import SymTridiagonal, gen_toeplitz
    out = {}
    for name in names:
        if name == "cfg1_uniform_N2000":
            rng = np.random.default_rng(0)
            a = rng.uniform(-1.0, 1.0, 2000)
            T = SymTridiagonal(a, rng.uniform(-1.0, 1.0, 1999))
            cfg = h.dc.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
        elif name == "cfg2_toeplitz_N10000_adc2":
            T = gen_toeplitz(10000)
            cfg = h.dc.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
        elif name == "cfg3_kac_N20000":
            i = np.arange(1, 20000, dtype=np.float64)
            T = SymTridiagonal(np.zeros(20000), np.sqrt(i * (20000 - i)))
            cfg = h.dc.SolverConfig(rank_eps=1e-13)
        else:
            continue
        t0 = time.perf_counter()
        h.dc.adc_solve(T, cfg)
        out[name] = {"wall_s": time.perf_counter() - t0, "cores": os.cpu_count(),
                     "kind": "reference"}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count()
    vals = []
    kind = "port"
    for i in range(args.warmup + args.steps):
        tf, dt, fl, kind = cpu_merge(CPU_SAMPLE_N)
        if i >= args.warmup:
            vals.append((tf, dt))
    tf = statistics.median(v[0] for v in vals)
    ms = statistics.median(v[1] for v in vals) * 1e3
    sample = (f"config-4 merge at N={CPU_SAMPLE_N} (the N = 32768 workload does not fit a "
              f"bounded CPU run: 173.6 s per merge on 8 cores); one merge per step: secular + "
              f"Loewner + normalizers + HSS construct + HSS x Q_old, "
              f"{'the reference itself (baseline/_ref)' if kind == 'reference' else 'oracle port'}"
              f", OpenBLAS threads = {threads}")
    line = {
        "impl": "reference", "metric": metric_name(), "value": tf, "unit": "TF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(CPU_SAMPLE_N, world),
        "cpu_baseline": {"value": tf, "unit": "TF/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": tf, "unit": "TF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name():
    return ("merge-step FP64 TF/s (the reference's FlopCounter work for the input / wall time; "
            "HSS eigvec-update incl. secular/Loewner/build/multiply)")


def config_dict(n, world):
    return {"workload": "config4_isolated_top_merge", "N": n, "leaf_size": LEAF,
            "rank_eps": RANK_EPS, "oversample": OVERSAMPLE, "id_tol": 1e-15, "rho": 1.0,
            "method": "adc-rand", "parallelism": f"rowblock{world}" if world > 1 else "single",
            "l2": (f"inputs larger than L2 (Q_old {n * n * 8 / 1e9:.1f} GB)" if n * n * 8 > 126e6
                   else f"Q_old {n * n * 8 / 1e6:.0f} MB fits L2 (126 MB)")}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- GPU arm
def measure_dgemm_peak(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    return 2 * n ** 3 / (e0.elapsed_time(e1) / 4 * 1e-3) / 1e12


def adc1_merge(d, u, rho, Q, out, reps=2):
    """Config-4 merge with ADC1 (method "adc-srrsc"): secular -> Loewner -> normalizers ->
    SRRSC construction -> HSS x Q_old, device-timed phase by phase (best of reps)."""
    import torch

    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200.flops import FlopCounter
    best = None
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        fl = FlopCounter()
        ev[0].record()
        sys_ = hb.RankOneSystem(d, u, rho)
        sol = hb.solve_secular(sys_, flops=fl)
        hb.recompute_weights(sys_.d, sol, sys_.z, rho=rho, flops=fl)
        C = hb.CauchyEvecMatrix.from_secular(sys_, sol, flops=fl)
        ev[1].record()
        part = hb.build_partition(C.k, 128, C.d, C.gamma, C.mu)
        H = hb.srrsc_hss_construct(C, part, hb.srrsc_cap(part), tol=1e-15, flops=fl)
        ev[2].record()
        if not H.flagged:
            hb.hss_matmul_right(Q, H, flops=fl, out=out)
        ev[3].record()
        torch.cuda.synchronize()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        rec = {"ms": sum(ms), "secular_loewner_normalizers_ms": ms[0], "construct_ms": ms[1],
               "multiply_ms": ms[2], "r_used": int(H.r_used), "flagged": bool(H.flagged),
               "flops": fl.as_dict()}
        if best is None or rec["ms"] < best["ms"]:
            best = rec
    return best


def _metrics_gpu(T, lam, Q, with_bwd=True):
    """orthogonality / backward / residual with the reference's formulas (cli.py:63-71)."""
    import torch
    n = T.n
    lam_d = torch.as_tensor(np.asarray(lam), device="cuda")
    G = Q.T @ Q
    G.diagonal().sub_(1.0)
    orth = float(G.abs().max()) / n
    del G
    bwd = None
    if with_bwd:
        A = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        i = torch.arange(n, device="cuda")
        A[i, i] = torch.as_tensor(T.a, device="cuda")
        A[i[:-1], i[1:]] = torch.as_tensor(T.b, device="cuda")
        A[i[1:], i[:-1]] = torch.as_tensor(T.b, device="cuda")
        A -= (Q * lam_d[None, :]) @ Q.T
        bwd = float(A.abs().max()) / (T.norm_max() * n)
        del A
    a = torch.as_tensor(T.a, device="cuda")
    b = torch.as_tensor(T.b, device="cuda")
    TQ = a[:, None] * Q
    TQ[:-1] += b[:, None] * Q[1:]
    TQ[1:] += b[:, None] * Q[:-1]
    resid = float((TQ - Q * lam_d[None, :]).abs().max()) / (n * T.norm_max())
    return orth, bwd, resid


def glue_gbs(T, cfg):
    """Achieved HBM GB/s of the glue kernels (blockdiag assembly + Givens replay, final
    column gather) over one full solve: algorithmic bytes / CUDA-event time per depth."""
    import torch

    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200 import solver
    solver.GLUE_PROFILE = []
    try:
        hb.adc_solve(T, cfg)
        torch.cuda.synchronize()
        prof = solver.GLUE_PROFILE
    finally:
        solver.GLUE_PROFILE = None
    out = {}
    for kind in ("assemble", "gather"):
        rows = [(e0.elapsed_time(e1), nb) for k, e0, e1, nb in prof if k == kind]
        ms = sum(r[0] for r in rows)
        nb = sum(r[1] for r in rows)
        out[kind] = {"ms": ms, "bytes": nb, "GB_s": nb / (ms * 1e-3) / 1e9 if ms else None}
    return out


def eigh_lines(peak_hbm=None):
    """Full tridiagonal eigendecompositions (BASELINE configs 1, 2, 3, 5) on one GPU: wall-s
    with Q left on the device, e2e wall-s with Q returned to pinned host memory (the
    reference's adc_solve returns a host Q, dc.py:65-79), the parity metrics with the
    reference's formulas and their ratio to the reference's own values on the same input
    (tests/golden/configs.npz, north_star's <= 10x rule), and the glue kernels' HBM GB/s
    (configs 1 and 5).  Config 2 is ADC1 as BASELINE names it (SRRSC construction, method
    "adc-srrsc"; no reference implementation exists) and, beside it, ADC2.
    """
    import torch

    import paper_1510_04591_b200 as hb
    gpath = os.path.join(ROOT, "tests", "golden", "configs.npz")
    g = np.load(gpath) if os.path.exists(gpath) else None
    out = {}
    toe = np.sort(2 + 2 * np.cos(np.arange(1, 10001) * np.pi / 10001))
    kac = -(20000 - 1) + 2.0 * np.arange(20000)
    cases = [  # name, T, cfg, exact spectrum, fixture tag, glue
        ("cfg1_uniform_N2000", hb.gen_uniform(2000, 0),
         hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13), None, "cfg1", True),
        ("cfg2_toeplitz_N10000_adc1", hb.gen_toeplitz(10000),
         hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13, method="adc-srrsc"),
         toe, None, False),
        ("cfg2_toeplitz_N10000_adc2", hb.gen_toeplitz(10000),
         hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13), toe, "cfg2r", False),
        ("cfg3_kac_N20000", hb.gen_kac(20000), hb.SolverConfig(rank_eps=1e-13), kac, "cfg3", False),
        ("cfg3_kac_N20000_defaults", hb.gen_kac(20000), hb.SolverConfig(), kac, "cfg3d", False),
        ("cfg5_N65536", hb.gen_config5(65536, 0), hb.SolverConfig(rank_eps=1e-13), None, None, True),
    ]
    import gc
    res = None
    for name, T, cfg, exact, tag, glue in cases:
        # the previous case's blocks are released first, so this case's warm-up leaves the
        # allocator holding exactly the segments its timed runs reuse
        res = None
        gc.collect()
        torch.cuda.empty_cache()
        hb.adc_solve(T, cfg)   # warm-up (allocator, tree buffers)
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = hb.adc_solve(T, cfg)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        n = T.n
        rec = {"wall_s": best, "method": cfg.method, "merges": len(res.merges),
               "hss_merges": int(sum(m.used_hss for m in res.merges)),
               "top_merge_hss": bool(res.merges[-1].used_hss)}
        if n <= 20000:
            # end to end as the reference API returns it: Q in (pinned) host memory
            hostQ = torch.empty(n, n, dtype=torch.float64, pin_memory=True)
            e2e = None
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r2 = hb.adc_solve(T, cfg)
                hostQ.copy_(r2.Q)
                dt = time.perf_counter() - t0
                e2e = dt if e2e is None else min(e2e, dt)
                del r2
            rec["wall_s_e2e"] = e2e
            rec["d2h_bytes"] = 8 * n * n
            del hostQ
        o, b, r = _metrics_gpu(T, res.lam, res.Q, with_bwd=n <= 20000)
        rec.update({"orthogonality": o, "backward": b, "residual": r})
        if exact is not None:
            rec["eig_err_over_normT"] = float(np.abs(res.lam - exact).max()) / T.norm_max()
        if g is not None and tag is not None and f"{tag}_orth" in g.files:
            ref = {m: float(g[f"{tag}_{m}"]) for m in ("orth", "bwd", "resid")}
            rec["reference"] = dict(ref, wall_s_survey_host=float(g[f"{tag}_wall_s"]))
            rec["ratio_to_reference"] = {"orthogonality": o / ref["orth"],
                                         "backward": (b / ref["bwd"]) if b is not None else None,
                                         "residual": r / ref["resid"]}
            rec["eig_err_vs_reference_over_normT"] = (
                float(np.abs(res.lam - g[f"{tag}_lam"]).max()) / T.norm_max())
        del res
        torch.cuda.empty_cache()
        if glue:
            gl = glue_gbs(T, cfg)
            if peak_hbm:
                for v in gl.values():
                    v["frac_of_hbm"] = v["GB_s"] / peak_hbm if v["GB_s"] else None
            rec["glue_hbm"] = gl
        out[name] = rec
        torch.cuda.empty_cache()
    return out


def eigh_distributed(world, ops=None, device="cuda", n=65536, warm=True):
    """BASELINE config 5 (N = 65536) solved across the torchrun ranks: subtrees per rank,
    row-block sharded top merges (distributed.adc_solve_distributed).  Wall-s is the max
    over ranks; orthogonality on 256 sampled columns, residual on every rank's rows."""
    import torch
    import torch.distributed as dist

    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200.distributed import GpuOps, adc_solve_distributed
    T = hb.gen_config5(n, 0)
    cfg = hb.SolverConfig(rank_eps=1e-13)
    ops = ops if ops is not None else GpuOps(4096)
    sync = torch.cuda.synchronize if device == "cuda" else (lambda: None)
    if warm:
        adc_solve_distributed(T, cfg, ops)      # warm-up: groups, allocator, buffers
    best = None
    for _ in range(2 if warm else 1):
        dist.barrier()
        sync()
        t0 = time.perf_counter()
        res = adc_solve_distributed(T, cfg, ops)
        sync()
        dt = torch.tensor([time.perf_counter() - t0], device=device)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        best = float(dt) if best is None else min(best, float(dt))
    Q = res.Q_rows
    r0, r1 = res.row0, res.row1
    lam = torch.as_tensor(res.lam, device=device)
    # residual of T Q - Q Lambda on this rank's rows (halo rows from the neighbours)
    edge = torch.stack([Q[0], Q[-1]])
    parts = [torch.empty_like(edge) for _ in range(world)]
    dist.all_gather(parts, edge)
    rk = dist.get_rank()
    a = torch.as_tensor(T.a[r0:r1], device=device)
    TQ = a[:, None] * Q
    bl = torch.as_tensor(T.b, device=device)
    TQ[:-1] += bl[r0:r1 - 1, None] * Q[1:]
    TQ[1:] += bl[r0:r1 - 1, None] * Q[:-1]
    if rk > 0:
        TQ[0] += bl[r0 - 1] * parts[rk - 1][1]
    if rk < world - 1:
        TQ[-1] += bl[r1 - 1] * parts[rk + 1][0]
    resid = torch.tensor([float((TQ - Q * lam[None, :]).abs().max())], device=device)
    del TQ
    dist.all_reduce(resid, op=dist.ReduceOp.MAX)
    ns = min(256, n)
    cols = torch.as_tensor(np.random.default_rng(0).choice(n, ns, replace=False), device=device)
    Gs = Q[:, cols].T @ Q
    dist.all_reduce(Gs)
    Gs[torch.arange(ns, device=device), cols] -= 1.0
    if hasattr(ops, "close"):
        ops.close()                # CUDA-IPC peer buffers unmapped in group order
    return {"wall_s": best, "ranks": world, "merges": len(res.merges),
            "hss_merges": int(sum(m.used_hss for m in res.merges)),
            "orthogonality_sampled_cols": ns, "orthogonality": float(Gs.abs().max()) / n,
            "residual": float(resid) / (n * T.norm_max())}


def reference_work(n):
    """The reference's FlopCounter for the config-4 merge at N = n on this exact input
    (secular + hss_construct + hss_mult over all n rows of Q_old), from the fixture the
    unmodified reference produced; None when not recorded for this N."""
    gp = os.path.join(ROOT, "tests", "golden", "configs.npz")
    tag = f"c4_{n}"
    if not os.path.exists(gp):
        return None
    g = np.load(gp)
    if f"{tag}_flops_mult_per_row" not in g.files:
        return None
    w = {"secular": int(g[f"{tag}_flops_secular"]), "hss_construct": int(g[f"{tag}_flops_construct"]),
         "hss_mult": int(g[f"{tag}_flops_mult_per_row"]) * n, "r_used": int(g[f"{tag}_r_used"])}
    w["total"] = w["secular"] + w["hss_construct"] + w["hss_mult"]
    return w


def nccl_summary(path):
    """NCCL version and the communicator lines of rank 0's NCCL_DEBUG=INFO log (init,
    transport / NVLS) for the bench line."""
    import torch
    out = {"version": ".".join(str(x) for x in torch.cuda.nccl.version())}
    if not path or not os.path.exists(path):
        return out
    lines = [ln.strip() for ln in open(path, errors="replace")]
    keep = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines
            if "NCCL INFO" in ln and any(t in ln for t in ("comm 0x", "NVLS", "via P2P", "nRanks",
                                                           "Channel 00", "CollNet", "Init COMPLETE"))]
    out["nvls"] = any("NVLS" in ln and ("enabled" in ln.lower() or "nvls comm" in ln.lower()
                                        or "support" in ln.lower()) for ln in lines)
    out["p2p_nvlink"] = any("P2P/CUMEM" in ln or "via P2P" in ln for ln in lines)
    out["lines"] = keep[:12]
    return out


def peak_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return None


def multiply_traffic():
    """DRAM bytes per multiply from the committed ncu capture, used only when it was taken
    on the multiply kernel source in this tree (sha256 of csrc/hss_mult.cu + tma.cuh)."""
    src = b"".join(open(os.path.join(ROOT, "paper_1510_04591_b200", "csrc", f), "rb").read()
                   for f in ("hss_mult.cu", "tma.cuh"))
    sha = hashlib.sha256(src).hexdigest()[:16]
    tp = os.path.join(ROOT, "profiles", "multiply_traffic.json")
    try:
        t = json.load(open(tp))
    except (OSError, ValueError):
        return None, "no ncu capture"
    if t.get("source_sha16") != sha:
        return None, f"profiles/multiply_traffic.json is from another kernel source ({t.get('source_sha16')})"
    return t.get("bytes_per_multiply"), f"profiles/multiply_traffic.json ({t.get('file')})"


def same_n_merge(n, cfg, args):
    """The GPU merge at the reference arm's sample size (device-resident, same protocol)."""
    import torch

    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200.merge_pipeline import MergePipeline
    d, u, rho = hb.isolated_merge_system(n, SEED)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    Q0, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen))
    Q0 = Q0.contiguous()                  # LAPACK order -> row-major rows for the multiply
    pipe = MergePipeline(n, cfg, rows=n)
    out = torch.empty_like(Q0)
    dd, uu = torch.as_tensor(d, device="cuda"), torch.as_tensor(u, device="cuda")
    for _ in range(max(3, args.warmup)):
        pipe.run(dd, uu, rho, Q0, seed=[SEED, 0], out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(5, args.steps)
    e0.record()
    for _ in range(steps):
        pipe.run(dd, uu, rho, Q0, seed=[SEED, 0], out=out)
    e1.record()
    torch.cuda.synchronize()
    return {"N": n, "ms_per_step": e0.elapsed_time(e1) / steps, "unit": "TF/s",
            "note": "value = the reference's flops for this input (cpu_baseline leg) / GPU time"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1510_04591_b200 as hb
    from paper_1510_04591_b200 import _native
    from paper_1510_04591_b200.merge_pipeline import MergePipeline

    rank, world, local = dist_env()
    # one rank per GPU; HSSEIG_DIST_BACKEND=gloo lets a one-GPU box run the N > 1 code path
    # (ranks share the device, host-side collectives) for testing
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1:
        backend = os.environ.get("HSSEIG_DIST_BACKEND", "nccl")
        if backend == "nccl" and "NCCL_DEBUG" not in os.environ:
            # communicator evidence (ranks, channels, NVLink / NVLS) into a per-rank file,
            # summarised in the JSON line; stdout stays one JSON line
            nccl_log = f"/tmp/hsseig_nccl.{os.getpid()}.log"
            os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,GRAPH,NVLS",
                              NCCL_DEBUG_FILE=nccl_log)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    lib = _native.load(build_if_missing=False)
    n = args.n
    d, u, rho = hb.isolated_merge_system(n, SEED)
    # Q_old: random orthogonal from the QR of a seeded Gaussian (setup, untimed)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    G = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    Q0, _ = torch.linalg.qr(G)
    del G
    r0, r1 = rank * n // world, (rank + 1) * n // world
    Qloc = Q0[r0:r1].contiguous()
    del Q0
    torch.cuda.empty_cache()
    cfg = hb.SolverConfig(leaf_size=LEAF, hss_threshold=4 * LEAF, rank_eps=RANK_EPS,
                          oversample=OVERSAMPLE, seed=SEED)
    d_dev = torch.as_tensor(d, device="cuda")
    u_dev = torch.as_tensor(u, device="cuda")
    if world == 1:
        pipe = MergePipeline(n, cfg, rows=r1 - r0)

        def step(Xin, out, dd=d_dev, uu=u_dev):
            return pipe.run(dd, uu, rho, Xin, seed=[SEED, 0], out=out)
    else:
        # row-block sharded merge: index-sharded roots / weights / samples + NCCL all-gathers
        from paper_1510_04591_b200.distributed import GpuOps, ShardedMerge
        sm = ShardedMerge(n, cfg, GpuOps(n))

        def step(Xin, out, dd=d_dev, uu=u_dev):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            lam, res, info = sm.run(dd, uu, rho, Xin, seed=[SEED, 0], rows_total=n)
            e1.record()
            out.copy_(res)
            torch.cuda.synchronize()
            tree = info["tree"]
            fl = dict(info["flops"])        # reference conventions over all n rows
            fl["hss_mult_local"] = (sm.ops.mult_flops(tree, Xin.shape[0])
                                    if info["used_hss"] else 0)
            ev = info.get("multiply_events")
            mult = ev[0].elapsed_time(ev[1]) if ev else float("nan")
            ms = {"total": e0.elapsed_time(e1), "multiply": mult}
            marks = info.get("marks") or []
            for (_, a), (name, b) in zip(marks, marks[1:]):   # device time per phase
                ms[name] = ms.get(name, 0.0) + a.elapsed_time(b) if name != "multiply" else mult
            return {"ms": ms,
                    "flops": fl,
                    "sample_gather": info.get("sample_gather"),
                    # dense work counted when the merge fell back (dc.py:132-138)
                    "flops_total_fullP": (fl["secular"] + fl["hss_construct"] + fl["hss_mult"]
                                          + fl["update_dense"]),
                    "r_used": info["r_used"], "used_hss": info["used_hss"]}

    out = torch.empty_like(Qloc)
    for _ in range(args.warmup):
        step(Qloc, out)
    torch.cuda.synchronize()
    peak = measure_dgemm_peak(torch) if rank == 0 else None

    # ---- device-resident timed region
    clk = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    launches0 = lib.hsseig_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    phase_ms = []
    e0.record()
    for _ in range(args.steps):
        info = step(Qloc, out)
        phase_ms.append(info)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    launches = lib.hsseig_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    rec = phase_ms[-1]
    flops_own = rec["flops_total_fullP"]     # one merge, all P rows, on OUR tree
    ref_work = reference_work(n)
    flops_total = ref_work["total"] if ref_work else flops_own
    value = flops_total / (ms * 1e-3) / 1e12
    mult_ms = statistics.median(p["ms"]["multiply"] for p in phase_ms)
    if not (mult_ms == mult_ms):   # no HSS multiply (dense fallback)
        mult_ms = ms
    mult_fl = rec["flops"]["hss_mult_local"]
    # the leaf up-level runs beside the construction on (SMs - reserve) CTAs: its SM-share
    # weighted time is the multiply's occupancy of the machine (reported beside the plain sum)
    leaf_ms = statistics.median(p["ms"].get("multiply_leaf_up", 0.0) for p in phase_ms)
    share = None
    if leaf_ms > 0:
        from paper_1510_04591_b200 import merge_pipeline as _mp
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        share = max(1, sms - _mp.SPLIT_RESERVE) / sms

    # ---- end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hQ = torch.empty(Qloc.shape, dtype=torch.float64, pin_memory=True)
        hQ.copy_(Qloc)
        hOut = torch.empty_like(hQ, pin_memory=True)
        hd = torch.as_tensor(d).pin_memory()
        hu = torch.as_tensor(u).pin_memory()
        Xd = torch.empty_like(Qloc)
        nst = max(2, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(nst):
            dd = hd.to("cuda", non_blocking=True)
            du = hu.to("cuda", non_blocking=True)
            if world == 1:
                # public streaming API: Q_old rows land in chunks while the factors are built,
                # Q_new rows go back while later chunks are multiplied
                pipe.run(dd, du, rho, Xd, seed=[SEED, 0], out=out, host_io=(hQ, hOut),
                         chunks=int(os.environ.get("HSSEIG_IO_CHUNKS", "16")))
            else:
                Xd.copy_(hQ, non_blocking=True)
                step(Xd, out, dd, du)
                hOut.copy_(out, non_blocking=True)
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / nst
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t)
        e2e = {"value": flops_total / (ems * 1e-3) / 1e12, "unit": "TF/s",
               "ms_per_step": ems,
               "h2d_bytes_per_step": int(hQ.numel() * 8 + 16 * n),
               "d2h_bytes_per_step": int(hOut.numel() * 8)}
        del hQ, hOut

    # ---- the same config-4 merge with ADC1 (SRRSC construction, no sample): informational
    adc1 = None
    if world == 1 and not args.no_eigh:
        adc1 = adc1_merge(d, u, rho, Qloc, out)

    # the full solves below need the HBM the merge bench holds (Q_old, outputs, workspaces)
    if world > 1:
        sm.ops.close()             # CUDA-IPC peer buffers unmapped in group order
    pipe = sm = step = Xd = None   # noqa: F841
    del Qloc, out
    import gc
    gc.collect()
    torch.cuda.empty_cache()

    eigh_d = None
    if world > 1 and not args.no_eigh and (world & (world - 1)) == 0:
        eigh_d = eigh_distributed(world)

    same_n = None
    if world == 1 and not args.no_cpu:
        same_n = same_n_merge(CPU_SAMPLE_N, cfg, args)

    if rank == 0:
        traffic, traffic_src = multiply_traffic()
        achieved = mult_fl / (mult_ms * 1e-3) / 1e12
        line = {
            "metric": metric_name(), "value": value, "unit": "TF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-4 system; Q_old = QR of a seeded Gaussian)",
            "config": dict(config_dict(n, world), **(
                {"sample_gather": "CUDA-IPC peer stores fused in the split-K reduction"
                 if rec.get("sample_gather") == "peer" else "NCCL all-gather"}
                if world > 1 else {})),
            "merge_wall_s": ms / 1e3,
            "phases_ms": {k: statistics.median(p["ms"][k] for p in phase_ms) for k in rec["ms"]},
            "flops_basis": ("reference FlopCounter on the reference's own tree for this input "
                            f"(tests/golden/configs.npz c4_{n})") if ref_work else
                           "FlopCounter conventions on our own tree (no reference count for this N)",
            "flops_reference": ref_work,
            "flops": rec["flops"], "value_own_tree": flops_own / (ms * 1e-3) / 1e12,
            "hss_rank": rec["r_used"], "used_hss": rec["used_hss"],
            "roofline": {"bound": "tensor", "kernel": "tma_gemm_kernel (HSS multiply, FP64 DMMA)",
                         "achieved": achieved, "peak": peak, "unit": "TF/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         **({"leaf_up_sm_share": share,
                             "achieved_sm_share_weighted": mult_fl / ((mult_ms - leaf_ms * (1 - share))
                                                                      * 1e-3) / 1e12,
                             "note": "the leaf up-level launch runs on a capped grid beside the "
                                     "construction (merge_pipeline.SPLIT_RESERVE SMs left to it); "
                                     "achieved counts its full duration"}
                            if share else {}),
                         "traffic_source": traffic_src,
                         "algorithmic": "multiply flops executed (our tree, reference counter "
                                        "conventions hss.py:329-357) / CUDA-event time of the "
                                        "multiply launches",
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64 entry)"},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if same_n is not None:
            line["same_n"] = same_n
        if world == 1 and not args.no_eigh:
            line["eigh"] = eigh_lines(peak_hbm())
            # the metric's HBM half: the full solve's HBM-bound kernel (final column gather of
            # every recursion depth of config 5) against the measured copy bandwidth
            gl = (line["eigh"].get("cfg5_N65536") or {}).get("glue_hbm") or {}
            ga = gl.get("gather")
            if ga and ga.get("GB_s"):
                pk = peak_hbm()
                line["roofline_hbm"] = {
                    "bound": "hbm", "kernel": "wave_gather_kernel<2, 4> (config 5, all depths)",
                    "achieved": ga["GB_s"], "peak": pk, "unit": "GB/s",
                    "frac": ga["GB_s"] / pk if pk else None, "traffic": None,
                    "algorithmic": "8 B written per output entry + 8 B read per kept entry and per "
                                   "own-child deflated entry (the other child's are structural zeros) "
                                   "/ CUDA-event time of the gather launches; ncu DRAM bytes per depth "
                                   "in profiles/round2_hbm_kernels.txt",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "unavailable"}
        if adc1 is not None:
            line["config4_adc1"] = adc1
        if world > 1 and eigh_d is not None:
            line["eigh"] = {"cfg5_N65536_distributed": eigh_d}
        if world > 1:
            line["nccl"] = nccl_summary(nccl_log)
        if not args.no_cpu and world == 1:
            tf, dt, fl, kind = cpu_merge(CPU_SAMPLE_N)
            line["cpu_baseline"] = {
                "value": tf, "unit": "TF/s", "cores": os.cpu_count(), "kind": kind,
                "sample": f"{'the reference (baseline/_ref)' if kind == 'reference' else 'oracle port'}"
                          f": config-4 merge at N={CPU_SAMPLE_N} ({dt:.2f} s, {fl:.3e} reference "
                          f"flops; OpenBLAS threads = host cores)"}
            if same_n is not None:
                same_n["value"] = fl / (same_n["ms_per_step"] * 1e-3) / 1e12
                same_n["ratio_to_cpu_reference"] = same_n["value"] / tf
            if not args.no_eigh:
                line["cpu_baseline"]["eigh"] = cpu_eigh(
                    ["cfg1_uniform_N2000", "cfg2_toeplitz_N10000_adc2"]
                    + (["cfg3_kac_N20000"] if args.cpu_eigh_all else []))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
