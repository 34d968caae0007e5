"""Secular roots, Loewner weights and column normalizers on the GPU.

Host mirror of pkg/src/hsseig/secular.py (same names, argument meaning and
exceptions).  Arrays live on the CUDA device as float64 torch tensors; numpy
inputs are uploaded.  Compute runs in libhsseig_b200.so (csrc/roots.cu).
"""
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .flops import secular_flops

EPS = float(np.finfo(np.float64).eps)


class SecularConvergenceError(ArithmeticError):
    """secular.py:25"""


class WeightRecomputationError(ArithmeticError):
    """secular.py:29"""


def dev_rows(x):
    """Row-major float64 device matrix; a CUDA view with unit column stride is kept as is."""
    if (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.ndim == 2
            and x.stride(1) == 1):
        return x
    return dev(x)


def dev(x, dtype=torch.float64):
    """Device float64 contiguous tensor view/copy of x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            x = x.to("cuda", non_blocking=False)
        return x.to(dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda").to(dtype)


class Status:
    """Device status block (hsseig_status) plus its host read-back."""

    def __init__(self, k):
        nat.require_cuda()
        # same initial state as hsseig_status_init, built with async device ops
        self.t = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.t[1:4] = int(k)

    def read(self):
        return self.t.cpu().tolist()


@dataclass
class RankOneSystem:
    """Post-deflation system diag(d) + rho z z^T (secular.py:33-57)."""

    d: object
    z: object
    rho: float

    def __post_init__(self):
        nat.require_cuda()
        self.d = dev(self.d)
        self.z = dev(self.z)
        if self.d.shape != self.z.shape or self.d.ndim != 1:
            raise ValueError("d and z must be 1-D arrays of equal length")
        if not (bool(torch.isfinite(self.d).all()) and bool(torch.isfinite(self.z).all())):
            raise ValueError("non-finite input")
        if not (self.rho > 0.0) or not np.isfinite(self.rho):
            raise ValueError("rho must be positive and finite")
        if self.size > 1 and bool((torch.diff(self.d) <= 0.0).any()):
            raise ValueError("poles must be strictly ascending")
        if self.size and bool((self.z == 0.0).any()):
            raise ValueError("zero weights must be deflated first")

    @property
    def size(self):
        return int(self.d.numel())


@dataclass
class SecularSolution:
    """Roots through gap pairs (secular.py:72-88); dnext carries the virtual pole."""

    lam: torch.Tensor
    gamma: torch.Tensor
    mu: torch.Tensor
    dnext: torch.Tensor | None = None
    zhat: torch.Tensor | None = None
    v: torch.Tensor | None = None
    iterations: int = 0
    iters: torch.Tensor | None = None

    @property
    def size(self):
        return int(self.lam.numel())

    @property
    def pole_bound(self):
        return float(self.lam[-1] + self.mu[-1])


EPS = float(np.finfo(np.float64).eps)


def deflation_tolerance(d, z, rho, eps_scale=1.0):
    """secular.py:91-93"""
    d = np.asarray(d, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    return eps_scale * 8.0 * EPS * max(float(np.abs(d).max()), rho * float(np.sum(z * z)))


@dataclass
class DeflationOutcome:
    """secular.py (DeflationOutcome): the kept system, the column permutation (kept first,
    then the deflated poles ascending), Givens rotations in the caller's indices."""

    kept: RankOneSystem
    permutation: np.ndarray
    rotations: list
    deflated_eigenvalues: list
    n_deflated: int
    tol: float


def deflate(d, z, rho, eps_scale=1.0):
    """Deflate negligible weights and (near-)equal pole pairs (secular.py:96-156).

    O(n) host work (the restated C routine of csrc/glue.cu, the same one the solver
    runs for every merge); the kept system is returned on the device.
    """
    d = np.ascontiguousarray(d, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    if d.shape != z.shape or d.ndim != 1 or d.size < 1:
        raise ValueError("d and z must be 1-D arrays of equal positive length")
    if not (np.all(np.isfinite(d)) and np.all(np.isfinite(z)) and np.isfinite(rho)):
        raise ValueError("non-finite input")
    if rho <= 0.0:
        raise ValueError("rho must be positive")
    n = d.size
    tol = deflation_tolerance(d, z, rho, eps_scale)
    d_out, z_out = np.empty(n), np.empty(n)
    perm = np.empty(n, dtype=np.int64)
    ri, rj = np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64)
    rc, rs = np.empty(n), np.empty(n)
    nrot = ctypes.c_int64(0)
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    k = int(nat.load().hsseig_deflate_tol(P(d), P(z), n, float(rho), float(tol), P(d_out), P(z_out),
                                          P(perm), P(ri), P(rj), P(rc), P(rs), ctypes.byref(nrot)))
    nr = int(nrot.value)
    rotations = [(int(ri[t]), int(rj[t]), float(rc[t]), float(rs[t])) for t in range(nr)]
    deflated = [(int(perm[t]), float(d_out[t])) for t in range(k, n)]
    kept = RankOneSystem(d_out[:k].copy(), z_out[:k].copy(), float(rho))
    return DeflationOutcome(kept=kept, permutation=perm.astype(np.intp), rotations=rotations,
                            deflated_eigenvalues=deflated, n_deflated=n - k, tol=tol)


def solve_secular(sys, flops=None, check=True):
    """All k roots (secular.py:159-180 over _kernels.pyx:178-234), one warp per 4 roots."""
    k = sys.size
    if k == 0:
        raise ValueError("empty system")
    lib = nat.load()
    lam = torch.empty(k, dtype=torch.float64, device="cuda")
    gam = torch.empty_like(lam)
    mu = torch.empty_like(lam)
    dn = torch.empty_like(lam)
    its = torch.empty(k, dtype=torch.int32, device="cuda")
    work = torch.empty(2 * k + 64, dtype=torch.float64, device="cuda")
    st = Status(k)
    s = nat.stream_ptr()
    nat.check(lib.hsseig_secular(nat.ptr(sys.d), nat.ptr(sys.z), k, float(sys.rho), nat.ptr(lam),
                                 nat.ptr(gam), nat.ptr(mu), nat.ptr(its), nat.ptr(work),
                                 nat.ptr(st.t), s), "secular")
    nat.check(lib.hsseig_dnext(nat.ptr(sys.d), nat.ptr(gam), nat.ptr(mu), k, nat.ptr(dn), s), "dnext")
    sol = SecularSolution(lam=lam, gamma=gam, mu=mu, dnext=dn, iters=its)
    sol._status = st
    if check:
        finish_secular(sol, k, flops)
    return sol


def finish_secular(sol, k, flops=None):
    """Read the status block: iteration total and the bracket check (secular.py:170-179)."""
    v = sol._status.read()
    sol.iterations = int(v[0])
    if flops is not None:
        flops.secular += secular_flops(k, sol.iterations)
    bad = v[1] if v[1] < k else (v[2] if (k >= 2 and v[2] < k) else -1)
    if bad >= 0:
        raise SecularConvergenceError(
            f"root {bad} lost its bracket (gamma={float(sol.gamma[bad]):.3e}, "
            f"mu={float(sol.mu[bad]):.3e})")
    return sol


def finish_secular_status_only(sol):
    """Iteration total without the bracket check (the raw kernel contract of secular_all)."""
    sol.iterations = int(sol._status.read()[0])
    return sol


def stable_gap(i, j, d, gamma, mu):
    """d[i] - lam[j] without cancellation (secular.py:183-192)."""
    if i <= j:
        return (d[i] - d[j]) - gamma[j]
    return (d[i] - d[j + 1]) + mu[j]


def gap_table(rows, cols, d, gamma, mu):
    """Dense d[rows] - lam[cols] via the stable branches (secular.py:195-203), on device."""
    d, gamma, mu = dev(d), dev(gamma), dev(mu)
    rows = torch.as_tensor(rows, dtype=torch.int64, device="cuda")
    cols = torch.as_tensor(cols, dtype=torch.int64, device="cuda")
    dext = torch.cat([d, (d[-1:] + gamma[-1:]) + mu[-1:]])
    di = d[rows][:, None]
    le = (di - d[cols][None, :]) - gamma[cols][None, :]
    gt = (di - dext[cols + 1][None, :]) + mu[cols][None, :]
    return torch.where(rows[:, None] <= cols[None, :], le, gt)


def recompute_weights(d, sol, orig_z, rho=1.0, flops=None, check=True):
    """Loewner weights (secular.py:206-236); fills sol.zhat and returns it."""
    d = dev(d)
    z = dev(orig_z)
    k = int(d.numel())
    if sol.dnext is None:
        sol.dnext = torch.empty_like(d)
        nat.check(nat.load().hsseig_dnext(nat.ptr(d), nat.ptr(sol.gamma), nat.ptr(sol.mu), k,
                                          nat.ptr(sol.dnext), nat.stream_ptr()), "dnext")
    zh = torch.empty_like(d)
    st = Status(k)
    nat.check(nat.load().hsseig_loewner(nat.ptr(d), nat.ptr(sol.dnext), nat.ptr(sol.gamma),
                                        nat.ptr(sol.mu), nat.ptr(z), k, float(rho), nat.ptr(zh),
                                        nat.ptr(st.t), nat.stream_ptr()), "loewner")
    if flops is not None:
        flops.secular += 8 * k * k
    sol.zhat = zh
    sol._wstatus = st
    if check:
        finish_weights(sol, k)
    return zh


def finish_weights(sol, k):
    v = sol._wstatus.read()
    if v[3] < k:
        raise WeightRecomputationError(
            f"non-positive radicand at index {v[3]}; interlacing must have failed")


def column_normalizers(d, gamma, mu, zhat, flops=None, dnext=None):
    """v_j = 1 / ||zhat ./ (d - lam_j)|| (secular.py:239-250)."""
    d, gamma, mu, zhat = dev(d), dev(gamma), dev(mu), dev(zhat)
    k = int(d.numel())
    lib = nat.load()
    s = nat.stream_ptr()
    if dnext is None:
        dnext = torch.empty_like(d)
        nat.check(lib.hsseig_dnext(nat.ptr(d), nat.ptr(gamma), nat.ptr(mu), k, nat.ptr(dnext), s),
                  "dnext")
    v = torch.empty_like(d)
    nat.check(lib.hsseig_normalizers(nat.ptr(d), nat.ptr(dnext), nat.ptr(gamma), nat.ptr(mu),
                                     nat.ptr(zhat), k, nat.ptr(v), s), "normalizers")
    if flops is not None:
        flops.secular += 6 * k * k
    return v
