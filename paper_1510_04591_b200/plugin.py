"""Reference-facing plugin surface (what hsseig would bind).

* ``secular_all(d, z, rho) -> (lam, gamma, mu, iters)`` — same contract as the
  reference's compiled kernel (pkg/src/hsseig/_kernels.pyx:178-234): NumPy in, NumPy
  out, outputs allocated by the callee.  Runs on the GPU.
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


def merge_update(Qk, d, z, rho, cfg, seed=0, flops=None, record=None):
    on_device = isinstance(Qk, torch.Tensor) and Qk.is_cuda
    lam, Qn, _ = _dc.merge_update(d, z, rho, Qk, cfg, seed=seed, flops=flops, record=record)
    if on_device:
        return lam, Qn
    return lam.cpu().numpy(), Qn.cpu().numpy()
