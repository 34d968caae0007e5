"""Shared test helpers: golden-fixture loading and seeded systems."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EPS = float(np.finfo(np.float64).eps)


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def random_system(rng, k, span=4.0, min_gap_frac=0.25, rho=None):
    """Jittered-grid poles, weights away from the deflation scale (pkg/tests/conftest.py:9-18)."""
    gap = span / k
    jitter = rng.uniform(-0.5 + min_gap_frac, 0.5 - min_gap_frac, k)
    d = (np.arange(k) + 0.5 + jitter) * gap
    z = rng.standard_normal(k)
    z[np.abs(z) < 0.05] += 0.1
    if rho is None:
        rho = 0.5 + rng.random()
    return d, z, float(rho)


def config4_system(n, seed):
    """BASELINE config 4: d_{i+1}-d_i ~ U(0.5,1.5)/N, u ~ N(0,1)/||u||, rho = 1."""
    rng = np.random.default_rng(seed)
    d = np.cumsum(rng.uniform(0.5, 1.5, n) / n)
    u = rng.standard_normal(n)
    u /= np.linalg.norm(u)
    return d, u, 1.0


def unpack_tree(g, prefix):
    """Per-node dicts from a packed reference tree (see golden/make_golden.py:pack_tree)."""
    meta = g[prefix + "meta"]
    out = []
    offs = {}
    for name in ("U", "V", "B", "rsel", "csel"):
        lens = g[f"{prefix}{name}_len"]
        offs[name] = (np.concatenate([[0], np.cumsum(lens)]), g[prefix + name])
    for i, (lo, hi, level, left, right, rU, rV, leaf) in enumerate(meta):
        nd = dict(lo=int(lo), hi=int(hi), level=int(level), left=int(left), right=int(right),
                  rU=int(rU), rV=int(rV), leaf=bool(leaf))
        for name in ("U", "V", "B", "rsel", "csel"):
            o, flat = offs[name]
            nd[name] = flat[o[i]:o[i + 1]]
        p = (hi - lo) if leaf else None
        if rU >= 0:
            rows = nd["U"].size // max(rU, 1) if rU else 0
            nd["U"] = nd["U"].reshape(rows, rU) if rU else nd["U"].reshape(-1, 0)
            nd["V"] = nd["V"].reshape(nd["V"].size // max(rV, 1), rV) if rV else nd["V"].reshape(-1, 0)
        out.append(nd)
    return out


def align_columns(Q, ref):
    s = np.sign((Q * ref).sum(axis=0))
    s[s == 0.0] = 1.0
    return Q * s
