"""Reference-facing plugin surface (what hsseig would bind).

* ``secular_all(d, z, rho) -> (lam, gamma, mu, iters)`` — same contract as the
  reference's compiled kernel (pkg/src/hsseig/_kernels.pyx:178-234): NumPy in, NumPy
  out, outputs allocated by the callee.  Runs on the GPU.
* ``tql2(d, e, Z, max_iter=30) -> int`` — the base-case kernel contract
  (_kernels.pyx:352-411, called by dc.py:118-129): in place on NumPy arrays, returns
  0 or 1 + the index of the eigenvalue whose QL iteration stalled.  Runs on the GPU
  (warp-per-matrix QL, n <= 32).  The eigenpairs come back in ascending order, which
  is the order the reference's caller sorts them into.
* ``merge_update(Qk, d, z, rho, cfg, seed, flops, record)`` — the merge body of
  dc.py:236-247 for one post-deflation system; returns (lam, Qk_new) as NumPy arrays
  (or torch CUDA tensors when Qk is one).
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
    Q = torch.empty(n * n, **dev)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.hsseig_tql2_batched(nat.ptr(a_d), nat.ptr(b_d), nat.ptr(off), 1, int(max_iter),
                                      nat.ptr(lam), nat.ptr(Q), nat.ptr(qoff), nat.ptr(st),
                                      nat.stream_ptr()), "tql2_batched")
    status = int(st.cpu()[0])
    if status:
        return status
    d[:] = lam.cpu().numpy()
    Zq = torch.as_tensor(np.ascontiguousarray(Z, dtype=np.float64), **dev) @ Q.view(n, n)
    Z[:, :] = Zq.cpu().numpy()
    e[:] = 0.0
    return 0


def merge_update(Qk, d, z, rho, cfg, seed=0, flops=None, record=None):
    on_device = isinstance(Qk, torch.Tensor) and Qk.is_cuda
    lam, Qn, _ = _dc.merge_update(d, z, rho, Qk, cfg, seed=seed, flops=flops, record=record)
    if on_device:
        return lam, Qn
    return lam.cpu().numpy(), Qn.cpu().numpy()
