"""Generator-held Cauchy-like eigenvector matrix on the GPU.

Mirror of pkg/src/hsseig/cauchy.py: C[i, j] = zhat[i] v[j] / (d[i] - lam[j]) is
never stored; blocks, products and the dense update generate tiles on the fly
in shared memory (csrc/cauchy.cu).
"""
import numpy as np
import torch

from . import _native as nat
from .flops import cauchy_eval_flops, gemm_flops
from .secular import column_normalizers, dev, dev_rows, stable_gap

MAX_SAMPLE_WIDTH = 128
DENSE_PANEL_MIN_K = 512           # below: the fused kernel (C tiles generated in smem)
DENSE_PANEL_BYTES = 2 << 30       # column panels of C materialised for the dense update


class CauchyEvecMatrix:
    """Square Cauchy-like matrix with unit columns (cauchy.py:15-27)."""

    def __init__(self, d, gamma, mu, zhat, v, dnext=None):
        self.d, self.gamma, self.mu = dev(d), dev(gamma), dev(mu)
        self.zhat, self.v = dev(zhat), dev(v)
        self.k = int(self.d.numel())
        if len({tuple(a.shape) for a in (self.d, self.gamma, self.mu, self.zhat, self.v)}) != 1:
            raise ValueError("generator arrays must share one shape")
        if dnext is None:
            dnext = torch.empty_like(self.d)
            nat.check(nat.load().hsseig_dnext(nat.ptr(self.d), nat.ptr(self.gamma),
                                              nat.ptr(self.mu), self.k, nat.ptr(dnext),
                                              nat.stream_ptr()), "dnext")
        self.dnext = dev(dnext)
        self._gen = nat.Gen(self.d.data_ptr(), self.dnext.data_ptr(), self.gamma.data_ptr(),
                            self.mu.data_ptr(), self.zhat.data_ptr(), self.v.data_ptr(), self.k)

    @classmethod
    def from_secular(cls, sys, sol, flops=None):
        """cauchy.py:29-38: computes v if not yet recorded."""
        if sol.zhat is None:
            raise ValueError("recompute_weights must run first")
        v = sol.v
        if v is None or bool(torch.isnan(v).any()):
            v = column_normalizers(sys.d, sol.gamma, sol.mu, sol.zhat, flops=flops, dnext=sol.dnext)
            sol.v = v
        return cls(sys.d, sol.gamma, sol.mu, sol.zhat, v, dnext=sol.dnext)

    @property
    def gen(self):
        return self._gen

    @property
    def lam(self):
        return self.d + self.gamma

    def entry(self, i, j):
        return float(self.zhat[i] * self.v[j] / stable_gap(i, j, self.d, self.gamma, self.mu))

    def _idx(self, r):
        if isinstance(r, (slice, range)):
            return torch.arange(self.k, device="cuda")[r]
        return torch.as_tensor(r, dtype=torch.int64, device="cuda").reshape(-1)

    def block(self, rows, cols, flops=None, phase="hss_construct"):
        """Dense C[rows, cols] (cauchy.py:48-56)."""
        rows, cols = self._idx(rows), self._idx(cols)
        out = torch.empty(rows.numel(), cols.numel(), dtype=torch.float64, device="cuda")
        if out.numel():
            nat.check(nat.load().hsseig_cauchy_block(self._gen, nat.ptr(rows), rows.numel(),
                                                     nat.ptr(cols), cols.numel(), nat.ptr(out),
                                                     cols.numel(), nat.stream_ptr()), "cauchy_block")
        if flops is not None:
            setattr(flops, phase, getattr(flops, phase) + cauchy_eval_flops(out.numel()))
        return out

    def to_dense(self, flops=None, phase="hss_construct"):
        idx = torch.arange(self.k, device="cuda")
        return self.block(idx, idx, flops=flops, phase=phase)

    def sample(self, omega, flops=None, phase="hss_construct", leaf_of=None):
        """(Y, Z) = (C @ Omega, C^T @ Omega) from one generator pass each (cauchy.py:70-100).

        leaf_of (device int32 per index, a tree's ``ct.leaf_of``): the off-diagonal sample
        instead, every leaf's diagonal block C(t, t) counted as zero (Y_t = Phi_t directly)."""
        omega = dev(omega)
        if omega.ndim != 2 or omega.shape[0] != self.k:
            raise ValueError(f"shape mismatch: C is {self.k}x{self.k}, Omega has {tuple(omega.shape)}")
        w = omega.shape[1]
        if w > MAX_SAMPLE_WIDTH:
            parts = [self.sample(omega[:, s:s + MAX_SAMPLE_WIDTH], leaf_of=leaf_of)
                     for s in range(0, w, MAX_SAMPLE_WIDTH)]
            Y, Z = torch.cat([p[0] for p in parts], 1), torch.cat([p[1] for p in parts], 1)
        else:
            lib = nat.load()
            if omega.stride(0) % 2 or omega.data_ptr() % 16:   # TMA wants 16-byte aligned rows
                padded = torch.zeros(self.k, w + (w % 2), dtype=torch.float64, device="cuda")
                padded[:, :w] = omega
                omega = padded
            Y = torch.empty(self.k, w, dtype=torch.float64, device="cuda")
            Z = torch.empty_like(Y)
            work = torch.empty(int(lib.hsseig_sample_work_doubles(self.k, w)), dtype=torch.float64,
                               device="cuda")
            nat.check(lib.hsseig_cauchy_sample(self._gen, leaf_of, nat.ptr(omega), omega.stride(0), w,
                                               nat.ptr(Y), nat.ptr(Z), w, nat.ptr(work),
                                               nat.stream_ptr()), "cauchy_sample")
        if flops is not None:
            each = gemm_flops(self.k, self.k, w) + cauchy_eval_flops(self.k * self.k)
            setattr(flops, phase, getattr(flops, phase) + 2 * each)
        return Y, Z

    def multiply(self, X, flops=None, phase="hss_construct"):
        """C @ X (cauchy.py:70-84)."""
        X = dev(X)
        vec = X.ndim == 1
        Y, _ = self.sample(X[:, None] if vec else X)
        if flops is not None:
            p = 1 if vec else X.shape[1]
            setattr(flops, phase, getattr(flops, phase) + gemm_flops(self.k, self.k, p)
                    + cauchy_eval_flops(self.k * self.k))
        return Y[:, 0] if vec else Y

    def transpose_multiply(self, X, flops=None, phase="hss_construct"):
        """C^T @ X (cauchy.py:86-100)."""
        X = dev(X)
        vec = X.ndim == 1
        _, Z = self.sample(X[:, None] if vec else X)
        if flops is not None:
            p = 1 if vec else X.shape[1]
            setattr(flops, phase, getattr(flops, phase) + gemm_flops(self.k, self.k, p)
                    + cauchy_eval_flops(self.k * self.k))
        return Z[:, 0] if vec else Z

    def right_multiply_into(self, Qblock, out=None):
        """out = Qblock @ C with C generated on the fly (dense update, dc.py:132-138)."""
        Q = dev_rows(Qblock)
        if Q.shape[1] != self.k:
            raise ValueError("inner dimensions do not match")
        if out is None:
            out = torch.empty(Q.shape[0], self.k, dtype=torch.float64, device="cuda")
        lib = nat.load()
        if self.k >= DENSE_PANEL_MIN_K and Q.shape[0] > 0:
            # materialised column panels of C (<= DENSE_PANEL_BYTES) on the TMA/DMMA engine
            if Q.stride(0) % 2 or Q.data_ptr() % 16:
                Qp = torch.empty(Q.shape[0], self.k + (self.k & 1), dtype=torch.float64, device="cuda")
                Qp[:, :self.k] = Q
                Q = Qp[:, :self.k]
            cols = max(128, DENSE_PANEL_BYTES // (8 * self.k))
            work = torch.empty(int(lib.hsseig_dense_update_work_doubles(self.k, cols)),
                               dtype=torch.float64, device="cuda")
            nat.check(lib.hsseig_dense_update_ws(nat.ptr(Q), Q.stride(0), Q.shape[0], self._gen,
                                                 nat.ptr(out), out.stride(0), nat.ptr(work),
                                                 work.numel(), nat.stream_ptr()), "dense_update")
            return out
        nat.check(lib.hsseig_dense_update(nat.ptr(Q), Q.stride(0), Q.shape[0], self._gen,
                                          nat.ptr(out), out.stride(0), nat.stream_ptr()),
                  "dense_update")
        return out

    def right_multiply_halves_into(self, W, n1, perm, ka, kb, out=None):
        """out = W @ C for W = the kept columns of a merge's blockdiag(Q1, Q2) block (rows
        [0, n1) from child 1): perm orders the kept columns [child 1 only | rotated | child 2
        only], the top rows contract over perm[:ka], the bottom rows over perm[kb:] -- the
        dense update (dc.py:132-138) without its products with structural zeros."""
        W = dev_rows(W)
        P, k = W.shape
        if k != self.k:
            raise ValueError("inner dimensions do not match")
        if W.stride(0) % 2 or W.data_ptr() % 16:
            raise ValueError("W rows must be 16-byte aligned (even leading dimension)")
        if out is None:
            out = torch.empty(P, k, dtype=torch.float64, device="cuda")
        lib = nat.load()
        perm_d = torch.as_tensor(np.ascontiguousarray(perm, dtype=np.int64), device="cuda")
        cols = max(128, DENSE_PANEL_BYTES // (8 * k))
        work = torch.empty(int(lib.hsseig_dense_update_halves_work_doubles(P, k, cols)),
                           dtype=torch.float64, device="cuda")
        nat.check(lib.hsseig_dense_update_halves(nat.ptr(W), W.stride(0), P, int(n1), self._gen,
                                                 nat.ptr(perm_d), int(ka), int(kb), nat.ptr(out),
                                                 out.stride(0), nat.ptr(work), work.numel(),
                                                 nat.stream_ptr()), "dense_update_halves")
        return out
