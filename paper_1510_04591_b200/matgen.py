"""Symmetric tridiagonal inputs (mirror of pkg/src/hsseig/matgen.py:17-112).

``SymTridiagonal(a, b)``: diagonal a (n), off-diagonal b (n-1), float64 on the host.
The generator families and their formulas follow the reference; the BASELINE
config generators (``gen_uniform``, ``gen_kac``, ``gen_config5``) draw d first,
then e, from ``np.random.default_rng(seed)``.
"""
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SymTridiagonal:
    a: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        a = np.ascontiguousarray(self.a, dtype=np.float64)
        b = np.ascontiguousarray(self.b, dtype=np.float64)
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b", b)
        if a.ndim != 1 or b.ndim != 1:
            raise ValueError("diagonals must be one-dimensional")
        if a.size < 1:
            raise ValueError("order must be at least 1")
        if b.size != a.size - 1:
            raise ValueError(f"need {a.size - 1} off-diagonal entries, got {b.size}")

    @property
    def n(self):
        return self.a.size

    def norm_max(self):
        m = float(np.abs(self.a).max())
        return max(m, float(np.abs(self.b).max())) if self.b.size else m

    def to_dense(self):
        A = np.diag(self.a)
        i = np.arange(self.n - 1)
        A[i, i + 1] = self.b
        A[i + 1, i] = self.b
        return A


def _order(n, minimum=1):
    if not isinstance(n, (int, np.integer)) or n < minimum:
        raise ValueError(f"order must be an integer >= {minimum}, got {n!r}")


def gen_clement(n):
    """b_i = sqrt(i (n+1-i)) (matgen.py:59-63)."""
    _order(n)
    i = np.arange(1, n, dtype=np.float64)
    return SymTridiagonal(np.zeros(n), np.sqrt(i * (n + 1 - i)))


def gen_legendre(n):
    _order(n, 2)
    i = np.arange(2, n + 1, dtype=np.float64)
    return SymTridiagonal(np.zeros(n), i / np.sqrt((2 * i - 1) * (2 * i + 1)))


def gen_laguerre(n):
    _order(n)
    return SymTridiagonal(2.0 * np.arange(1, n + 1) + 1.0, np.arange(2, n + 1, dtype=np.float64))


def gen_hermite(n):
    _order(n)
    return SymTridiagonal(np.zeros(n), np.sqrt(np.arange(1, n, dtype=np.float64)))


def gen_toeplitz(n):
    """a = 2, b = 1; eigenvalues 2 + 2 cos(j pi / (n+1))."""
    _order(n)
    return SymTridiagonal(np.full(n, 2.0), np.ones(n - 1))


def gen_kac(n):
    """BASELINE config 3: a = 0, b_i = sqrt(i (N - i)); eigenvalues -(N-1) + 2j."""
    _order(n)
    i = np.arange(1, n, dtype=np.float64)
    return SymTridiagonal(np.zeros(n), np.sqrt(i * (n - i)))


def gen_uniform(n, seed=0):
    """BASELINE config 1: a, b i.i.d. U(-1, 1), a drawn first."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, n)
    return SymTridiagonal(a, rng.uniform(-1.0, 1.0, n - 1))


def gen_config5(n, seed=0):
    """BASELINE config 5: a ~ U(0, 1), b ~ U(0.5, 1), a drawn first."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, n)
    return SymTridiagonal(a, rng.uniform(0.5, 1.0, n - 1))


def isolated_merge_system(n, seed=0):
    """BASELINE config 4 rank-one system: gaps U(0.5,1.5)/N, u ~ N(0,1)/||u||, rho = 1."""
    rng = np.random.default_rng(seed)
    d = np.cumsum(rng.uniform(0.5, 1.5, n) / n)
    u = rng.standard_normal(n)
    u /= np.linalg.norm(u)
    return d, u, 1.0


def uniform_pole_system(n, lo=1.0, hi=9.0, seed=0):
    """Example-1 system of the paper (matgen.py:102-112)."""
    d = np.arange(1, n + 1, dtype=np.float64) * ((hi - lo) / n)
    u = np.random.default_rng(seed).standard_normal(n)
    return d, u / np.linalg.norm(u)


FAMILIES = {
    "clement": gen_clement,
    "legendre": gen_legendre,
    "laguerre": gen_laguerre,
    "hermite": gen_hermite,
    "toeplitz": gen_toeplitz,
    "kac": gen_kac,
}
