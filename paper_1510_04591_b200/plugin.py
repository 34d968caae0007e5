"""Reference-facing plugin surface (what hsseig would bind).

* ``secular_all(d, z, rho) -> (lam, gamma, mu, iters)`` — same contract as the
  reference's compiled kernel (pkg/src/hsseig/_kernels.pyx:178-234): NumPy in, NumPy
  out, outputs allocated by the callee.  Runs on the GPU.
* ``tql2(d, e, Z, max_iter=30) -> int`` — the base-case kernel contract
  (_kernels.pyx:352-411, called by dc.py:118-129): in place on NumPy arrays (d and Z
  rotated in QL order, e untouched), returns 0 or 1 + the index of the eigenvalue whose
  QL iteration stalled.  Runs on the GPU (warp-per-matrix QL for n <= 32, a block per
  matrix up to n = 160); the caller's Z is the initial accumulator, as in the reference.
* ``merge_update(Qk, d, z, rho, cfg, seed, flops, record)`` — the merge body of
  dc.py:236-247 for one post-deflation system; returns (lam, Qk_new) as NumPy arrays
  (or torch CUDA tensors when Qk is one).
* ``update_vectors_hss(Qblock, C, cfg, seed, flops, record)`` and
  ``update_vectors_dense(Qblock, Qprime, flops)`` — drop-ins for the reference's own
  functions of the same names (dc.py:132-171), called with the REFERENCE's objects (its
  ``CauchyEvecMatrix`` generators, ``SolverConfig``, ``FlopCounter``, ``MergeRecord``),
  NumPy in / NumPy out: rebinding ``hsseig.dc.update_vectors_hss`` /
  ``update_vectors_dense`` routes the update branch of ``_solve_rec`` (dc.py:241-246) to
  the GPU with no other change to the reference.
* ``kernels()`` — a kernel namespace for ``hsseig.backend`` (``secular_all`` and
  ``tql2`` on the GPU; the reference's own Jacobi oracle kernels passed through).
"""
import numpy as np
import torch

from . import dc as _dc
from . import secular as _sec


def secular_all(d, z, rho):
    sys = _sec.RankOneSystem(np.ascontiguousarray(d, dtype=np.float64),
                             np.ascontiguousarray(z, dtype=np.float64), float(rho))
    sol = _sec.solve_secular(sys, check=False)
    _sec.finish_secular_status_only(sol)
    return (sol.lam.cpu().numpy(), sol.gamma.cpu().numpy(), sol.mu.cpu().numpy(),
            int(sol.iterations))


def tql2(d, e, Z, max_iter=30):
    """QL kernel contract of _kernels.pyx:352-411 / _kernels_py.py:300-360, run on the GPU:
    d (n) in/out in QL order (unsorted), e read only (the reference iterates on a copy), Z
    (any number of rows, n columns) rotated in place; returns 0 or 1 + the index of the
    eigenvalue that stalled (d / Z as far as the iteration got)."""
    from . import _native as nat
    from .solver import MAX_BASE
    n = d.shape[0]
    if n > MAX_BASE:
        raise ValueError(f"device QL handles base cases up to n = {MAX_BASE}")
    if e.shape[0] < n - 1 or Z.ndim != 2 or Z.shape[1] != n:
        raise ValueError("tql2 needs e of length >= n-1 and Z with n columns")
    if n <= 1:
        return 0
    nat.require_cuda()
    lib = nat.load()
    dev = dict(dtype=torch.float64, device="cuda")
    a_d = torch.as_tensor(np.ascontiguousarray(d, dtype=np.float64), **dev)
    b_d = torch.as_tensor(np.concatenate([np.asarray(e[:n - 1], dtype=np.float64), [0.0]]), **dev)
    off = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    qoff = torch.tensor([0, n * n], dtype=torch.int64, device="cuda")
    lam = torch.empty(n, **dev)
    square = Z.shape[0] == n
    # a square Z is the accumulator itself, rotated in place in the reference's order
    # (flag 1); otherwise the kernel accumulates from the identity and Z <- Z Q after
    Q = (torch.as_tensor(np.ascontiguousarray(Z, dtype=np.float64).ravel(), **dev).clone()
         if square else torch.empty(n * n, **dev))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.hsseig_tql2_batched(nat.ptr(a_d), nat.ptr(b_d), nat.ptr(off), 1, n, int(max_iter),
                                      nat.ptr(lam), nat.ptr(Q), nat.ptr(qoff), nat.ptr(st),
                                      3 if square else 2, nat.stream_ptr()), "tql2_batched")
    d[:] = lam.cpu().numpy()
    if square:
        Z[:, :] = Q.view(n, n).cpu().numpy()
    elif Z.shape[0]:
        ne = n + (n & 1)                      # TMA rows: even leading dimensions
        R = Z.shape[0]
        Zin = torch.zeros(R, ne, **dev)
        Zin[:, :n] = torch.as_tensor(np.asarray(Z, dtype=np.float64), **dev)
        Qp = torch.zeros(n, ne, **dev)
        Qp[:, :n] = Q.view(n, n)
        Zout = torch.empty(R, ne, **dev)
        nat.check(lib.hsseig_gemm(nat.ptr(Zin), ne, nat.ptr(Qp), ne, nat.ptr(Zout), ne, R, n, n,
                                  nat.stream_ptr()), "gemm")
        Z[:, :] = Zout[:, :n].cpu().numpy()
    return int(st.cpu()[0])


def merge_update(Qk, d, z, rho, cfg, seed=0, flops=None, record=None):
    on_device = isinstance(Qk, torch.Tensor) and Qk.is_cuda
    lam, Qn, _ = _dc.merge_update(d, z, rho, Qk, cfg, seed=seed, flops=flops, record=record)
    if on_device:
        return lam, Qn
    return lam.cpu().numpy(), Qn.cpu().numpy()


def _cfg(cfg):
    """The reference's SolverConfig (or any object with its fields) as ours."""
    return _dc.SolverConfig(**{f: getattr(cfg, f) for f in
                               ("base_size", "hss_threshold", "leaf_size", "oversample",
                                "rank_eps", "rank_cap", "seed", "method")})


def update_vectors_hss(Qblock, C, cfg, seed=0, flops=None, record=None):
    """dc.py:141-171 on the GPU for the reference's own arguments: C is the reference's
    CauchyEvecMatrix (its generators d, gamma, mu, zhat, v are uploaded; tiles, sample,
    construction and the multiply run in libhsseig_b200.so), cfg / flops / record are the
    reference's objects (fields updated in place with its conventions).  NumPy out."""
    from .cauchy import CauchyEvecMatrix
    Cd = CauchyEvecMatrix(C.d, C.gamma, C.mu, C.zhat, C.v)
    Q = torch.as_tensor(np.ascontiguousarray(Qblock, dtype=np.float64), device="cuda")
    out = _dc.update_vectors_hss(Q, Cd, _cfg(cfg), seed=seed, flops=flops, record=record)
    return out.cpu().numpy()


def update_vectors_dense(Qblock, Qprime, flops=None):
    """dc.py:132-138 on the GPU (FP64 DMMA GEMM) for NumPy operands; NumPy out."""
    Qb = np.asarray(Qblock)
    Qp = np.asarray(Qprime)
    if Qb.shape[1] != Qp.shape[0]:
        raise ValueError("inner dimensions do not match")
    out = _dc.update_vectors_dense(torch.as_tensor(np.ascontiguousarray(Qb, dtype=np.float64),
                                                   device="cuda"),
                                   torch.as_tensor(np.ascontiguousarray(Qp, dtype=np.float64),
                                                   device="cuda"), flops=flops)
    return out.cpu().numpy()


def kernels(reference_kernels=None):
    """Kernel namespace for hsseig.backend.load_kernels (backend.py:9-17): the GPU
    secular_all / tql2, and the reference's Jacobi kernels (its test oracle) passed
    through from `reference_kernels` when given."""
    import types
    ns = types.SimpleNamespace(secular_all=secular_all, tql2=tql2)
    if reference_kernels is not None:
        for name in ("jacobi_run", "onesided_orthogonalize"):
            if hasattr(reference_kernels, name):
                setattr(ns, name, getattr(reference_kernels, name))
    return ns
