"""Merge-step drivers and solver configuration (host mirror of pkg/src/hsseig/dc.py).

``update_vectors_dense`` / ``update_vectors_hss`` keep the reference signatures
and fallback rules (dc.py:132-171); ``merge_update`` is the merge body of
dc.py:236-247 (secular -> Loewner -> normalizers -> dense or HSS update) for one
post-deflation rank-one system whose eigenvector block already sits on the GPU.
"""
from dataclasses import dataclass, field

import os

import numpy as np
import torch

from .cauchy import DENSE_PANEL_MIN_K, CauchyEvecMatrix
from .flops import FlopCounter, cauchy_eval_flops, gemm_flops
from .hss import (DEFAULT_ID_TOL, MAX_WIDTH, build_partition, draw_omegas, estimate_rank,
                  finish_construct, hss_matmul_right, rand_hss_construct, srrsc_hss_construct)
from .secular import RankOneSystem, dev, dev_rows, recompute_weights, solve_secular

# "adc-srrsc" (ADC1) is named by BASELINE.json but absent from the reference (dc.py:23 knows
# the other two); its HSS construction is the SRRSC of oracle/srrsc_oracle.py
METHODS = ("dense-dc", "adc-rand", "adc-srrsc")
HSS_METHODS = ("adc-rand", "adc-srrsc")
SAMPLE_MODES = ("offdiag", "reference")


class BaseCaseError(ArithmeticError):
    """dc.py:27"""


@dataclass
class SolverConfig:
    """dc.py:30-51 (same fields, defaults and validation)."""

    base_size: int = 25
    hss_threshold: int = 2000
    leaf_size: int = 200
    oversample: int = 10
    rank_eps: float = 1e-16
    rank_cap: int = 100
    seed: int = 0
    method: str = "adc-rand"
    # ADC1 only: Schur-complement truncation max|S| <= srrsc_tol * max|block| (the
    # reference's ID truncation tolerance, hss.py:23); the rank cap is the smallest leaf
    srrsc_tol: float = DEFAULT_ID_TOL
    # ADC2 only: "offdiag" forms the leaves' Phi / Theta from the off-diagonal sample
    # C(t, t^c) Omega(t^c) (no cancellation against D Omega_t: half the ranks and a smaller
    # HSS error); "reference" is the reference's Y_t - D_t Omega_t
    sample: str = "offdiag"

    def __post_init__(self):
        if self.base_size < 3:
            raise ValueError("base_size must be at least 3")
        if self.hss_threshold < 4 * self.leaf_size:
            raise ValueError("hss_threshold must be at least 4x leaf_size")
        if self.rank_eps <= 0.0 or not (0 < self.rank_cap):
            raise ValueError("tolerances must be positive")
        if self.oversample < 0:
            raise ValueError("oversample must be non-negative")
        if self.method not in METHODS:
            raise ValueError(f"method must be one of {METHODS}")
        if not self.srrsc_tol >= 0.0:
            raise ValueError("srrsc_tol must be non-negative")
        if self.sample not in SAMPLE_MODES:
            raise ValueError(f"sample must be one of {SAMPLE_MODES}")


def split(T, k=None):
    """T = blockdiag(T1, T2) + rho v v^T, v = e_k + theta e_{k+1} (dc.py:82-102).

    rho = |b_k|, theta = sign(b_k): both corner diagonals drop by rho.  The level-batched
    solver applies the same arithmetic to every node of the recursion (solver._plan)."""
    from .matgen import SymTridiagonal
    n = T.n
    if k is None:
        k = n // 2
    if not 1 <= k < n:
        raise ValueError(f"split index {k} out of range for order {n}")
    bk = float(T.b[k - 1])
    rho = abs(bk)
    theta = 1.0 if bk >= 0.0 else -1.0
    a1 = T.a[:k].copy()
    a1[-1] -= rho
    a2 = T.a[k:].copy()
    a2[0] -= rho
    return SymTridiagonal(a1, T.b[:k - 1].copy()), SymTridiagonal(a2, T.b[k:].copy()), rho, theta


@dataclass
class MergeRecord:
    """dc.py:54-62"""

    size: int
    kept: int
    n_deflated: int
    used_hss: bool = False
    hss_rank: int = 0
    fell_back: bool = False
    flops: dict = field(default_factory=dict)


@dataclass
class EigenResult:
    """dc.py:65-79; lam and Q stay on the device (torch float64)."""

    lam: torch.Tensor
    Q: torch.Tensor
    merges: list = field(default_factory=list)
    flops: FlopCounter = field(default_factory=FlopCounter)

    @property
    def n(self):
        return int(self.lam.numel())

    def max_deflation_fraction(self):
        if not self.merges:
            return 0.0
        return max(m.n_deflated / m.size for m in self.merges)


def update_vectors_dense(Qblock, Qprime, flops=None, out=None):
    """Plain update Qblock @ Qprime (dc.py:132-138).

    Qprime may be a CauchyEvecMatrix: its tiles are then generated on the fly inside
    the DMMA GEMM (the reference first materialises C.to_dense(), counted the same way).
    """
    Qb = dev_rows(Qblock)
    if isinstance(Qprime, CauchyEvecMatrix):
        if Qb.shape[1] != Qprime.k:
            raise ValueError("inner dimensions do not match")
        if flops is not None:
            flops.update_dense += cauchy_eval_flops(Qprime.k * Qprime.k)
            flops.update_dense += gemm_flops(Qb.shape[0], Qprime.k, Qprime.k)
        return Qprime.right_multiply_into(Qb, out=out)
    from . import _native as nat
    Qp = dev(Qprime)
    if Qb.shape[1] != Qp.shape[0]:
        raise ValueError("inner dimensions do not match")
    if flops is not None:
        flops.update_dense += gemm_flops(Qb.shape[0], *Qp.shape)
    if out is None:
        out = torch.empty(Qb.shape[0], Qp.shape[1], dtype=torch.float64, device="cuda")
    # the TMA engine wants 16-byte aligned rows (even leading dimensions)
    if Qb.stride(0) % 2:
        Qb = torch.nn.functional.pad(Qb, (0, 1))[:, :Qb.shape[1]]
    if Qp.stride(0) % 2:
        Qp = torch.nn.functional.pad(Qp, (0, 1))[:, :Qp.shape[1]]
    nat.check(nat.load().hsseig_gemm(nat.ptr(Qb), Qb.stride(0), nat.ptr(Qp), Qp.stride(0),
                                     nat.ptr(out), out.stride(0), Qb.shape[0], Qp.shape[1],
                                     Qb.shape[1], nat.stream_ptr()), "gemm")
    return out


def srrsc_cap(part):
    """ADC1 rank cap: the smallest leaf (a node of that rank is not compressed at all)."""
    return min(part.min_leaf, MAX_WIDTH)


def update_vectors_hss(Qblock, C, cfg, seed=0, flops=None, record=None, omega=None,
                       return_tree=False):
    """HSS update with the reference's dense fallbacks (dc.py:141-171)."""
    k = C.k

    def dense_fallback():
        if record is not None:
            record.used_hss = False
            record.fell_back = True
        out = update_vectors_dense(Qblock, C, flops=flops)
        return (out, None) if return_tree else out

    try:
        part = build_partition(k, cfg.leaf_size, C.d, C.gamma, C.mu)
    except ValueError:
        return dense_fallback()
    if cfg.method == "adc-srrsc":
        H = srrsc_hss_construct(C, part, srrsc_cap(part), tol=cfg.srrsc_tol, flops=flops)
    else:
        r_est = estimate_rank(part, C.d, C.gamma, C.mu, cfg.rank_eps, cfg.rank_cap)
        r = min(r_est, part.min_leaf - cfg.oversample)
        if r < 1 or r + cfg.oversample > MAX_WIDTH:
            return dense_fallback()
        H = rand_hss_construct(C, part, r, p=cfg.oversample, seed=seed, flops=flops, omega=omega,
                               offdiag=cfg.sample == "offdiag")
    if H.flagged:
        return dense_fallback()
    if record is not None:
        record.used_hss = True
        record.hss_rank = H.r_used
    out = hss_matmul_right(Qblock, H, flops=flops)
    return (out, H) if return_tree else out


@dataclass
class HssJob:
    """One update_vectors_hss call of a batch: Qblock, C, seed, flops, record as there;
    d / gamma / mu are the host copies of C's generators (partition and rank estimate),
    out receives Qblock @ Q'."""
    Q: object
    C: object
    seed: object
    flops: object
    record: object
    d: np.ndarray
    gamma: np.ndarray
    mu: np.ndarray
    out: object
    # (n1, perm, ka, kb) when Q is the kept block of blockdiag(Q1, Q2): a dense fallback then
    # skips the structural zeros (CauchyEvecMatrix.right_multiply_halves_into)
    halves: object = None


_SIDE = []


def _side_streams(n):
    while len(_SIDE) < n:
        _SIDE.append(torch.cuda.Stream())
    return _SIDE[:n]


def update_vectors_hss_many(jobs, cfg, max_streams=None):
    """update_vectors_hss (dc.py:141-171) for every HSS merge of one recursion level.

    Phase by phase, so the level pays a handful of host waits instead of ~9 per merge
    (host partitions / rank estimates, every Gaussian draw, every sample + construction,
    then the multiplies), and merge i runs on side stream i mod max_streams so the
    latency-bound small kernels (interpolative decompositions, tree levels) of different
    merges overlap on the GPU.  Per job the operations and their inputs are exactly those
    of update_vectors_hss.  The caller's stream waits for all of it before returning.
    """
    if max_streams is None:
        max_streams = int(os.environ.get("HSSEIG_HSS_STREAMS", "8"))
    main = torch.cuda.current_stream()

    def dense_fallback(j):
        j.record.used_hss = False
        j.record.fell_back = True
        if j.halves is not None and j.C.k >= DENSE_PANEL_MIN_K:
            # same count as update_vectors_dense (the reference's, dc.py:132-138)
            j.flops.update_dense += cauchy_eval_flops(j.C.k * j.C.k) + gemm_flops(j.Q.shape[0], j.C.k, j.C.k)
            n1, perm, ka, kb = j.halves
            j.C.right_multiply_halves_into(j.Q, n1, perm, ka, kb, out=j.out)
            return
        j.out.copy_(update_vectors_dense(j.Q, j.C, flops=j.flops))

    live = []
    for j in jobs:
        try:
            part = build_partition(j.C.k, cfg.leaf_size, j.d, j.gamma, j.mu)
        except ValueError:
            dense_fallback(j)
            continue
        if cfg.method == "adc-srrsc":
            live.append((j, part, srrsc_cap(part)))
            continue
        r_est = estimate_rank(part, j.d, j.gamma, j.mu, cfg.rank_eps, cfg.rank_cap)
        r = min(r_est, part.min_leaf - cfg.oversample)
        if r < 1 or r + cfg.oversample > MAX_WIDTH:
            dense_fallback(j)
            continue
        live.append((j, part, r))
    if not live:
        return
    side = _side_streams(min(len(live), max_streams))
    for s in side:
        s.wait_stream(main)
    st = [side[i % len(side)] for i in range(len(live))]
    trees = []
    if cfg.method == "adc-srrsc":
        for (j, part, cap), s in zip(live, st):
            with torch.cuda.stream(s):
                trees.append(srrsc_hss_construct(j.C, part, cap, tol=cfg.srrsc_tol, finish=False))
    else:
        oms = draw_omegas([(j.C.k, r + cfg.oversample, j.seed) for j, _, r in live], streams=st)
        for (j, part, r), om, s in zip(live, oms, st):
            with torch.cuda.stream(s):
                trees.append(rand_hss_construct(j.C, part, r, p=cfg.oversample, seed=j.seed,
                                                omega=om, finish=False,
                                                offdiag=cfg.sample == "offdiag"))
        del oms
    for (j, _, _), H, s in zip(live, trees, st):
        with torch.cuda.stream(s):
            finish_construct(H, j.flops)
            if H.flagged:
                dense_fallback(j)
                continue
            j.record.used_hss = True
            j.record.hss_rank = H.r_used
            j.out.copy_(hss_matmul_right(j.Q, H, flops=j.flops))
    for s in side:
        main.wait_stream(s)


def merge_update(d, z, rho, Qblock, cfg, seed=0, flops=None, record=None, omega=None):
    """Merge body for one rank-one system (dc.py:236-247): returns (lam, Q_new, C)."""
    sys = RankOneSystem(d, z, rho)
    sol = solve_secular(sys, flops=flops)
    recompute_weights(sys.d, sol, sys.z, rho=rho, flops=flops)
    C = CauchyEvecMatrix.from_secular(sys, sol, flops=flops)
    if cfg.method in HSS_METHODS and sys.size > cfg.hss_threshold:
        Qn = update_vectors_hss(Qblock, C, cfg, seed=seed, flops=flops, record=record, omega=omega)
    else:
        Qn = update_vectors_dense(Qblock, C, flops=flops)
    return sol.lam, Qn, C
