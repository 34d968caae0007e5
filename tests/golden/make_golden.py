"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container only (it needs /root/reference):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to /tmp/hsseig_ref, builds the Cython extension
there (the reference's own setup.py, unmodified sources), imports ``hsseig`` and
writes small .npz fixtures next to this script.  The fixtures are committed; the
GPU box never reads /root/reference.
"""
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
BUILD = "/tmp/hsseig_ref"


def _import_reference():
    if not os.path.exists(os.path.join(BUILD, "src", "hsseig")):
        shutil.copytree(REF, BUILD)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=BUILD,
                   check=True, capture_output=True)
    sys.path.insert(0, os.path.join(BUILD, "src"))
    import hsseig  # noqa: F401
    assert hsseig.BACKEND == "c", hsseig.BACKEND
    return hsseig


def random_system(rng, k, span=4.0, min_gap_frac=0.25, rho=None):
    # same construction as the reference's conftest fixture (pkg/tests/conftest.py:9-18)
    gap = span / k
    jitter = rng.uniform(-0.5 + min_gap_frac, 0.5 - min_gap_frac, k)
    d = (np.arange(k) + 0.5 + jitter) * gap
    z = rng.standard_normal(k)
    z[np.abs(z) < 0.05] += 0.1
    if rho is None:
        rho = 0.5 + rng.random()
    return d, z, float(rho)


def config4_system(n, seed):
    # BASELINE config 4 shape: sorted poles with U(0.5,1.5)/N gaps, unit Gaussian u, rho=1
    rng = np.random.default_rng(seed)
    d = np.cumsum(rng.uniform(0.5, 1.5, n) / n)
    u = rng.standard_normal(n)
    u /= np.linalg.norm(u)
    return d, u, 1.0


def pack_tree(H, prefix, out):
    """Flatten an HssTree into arrays (postorder node index = reference node.index)."""
    nn = len(H.nodes)
    meta = np.zeros((nn, 8), dtype=np.int64)  # lo, hi, level, left, right, rU, rV, leaf
    U, V, B, D, RS, CS = [], [], [], [], [], []
    for nd in H.nodes:
        rU = nd.U.shape[1] if nd.U is not None else -1
        rV = nd.V.shape[1] if nd.V is not None else -1
        meta[nd.index] = (nd.lo, nd.hi, nd.level, nd.left, nd.right, rU, rV, int(nd.is_leaf))
        U.append(nd.U.ravel() if nd.U is not None else np.zeros(0))
        V.append(nd.V.ravel() if nd.V is not None else np.zeros(0))
        B.append(nd.B.ravel() if nd.B is not None else np.zeros(0))
        D.append(nd.D.ravel() if nd.D is not None else np.zeros(0))
        RS.append(nd.rows_sel if nd.rows_sel is not None else np.zeros(0, dtype=np.intp))
        CS.append(nd.cols_sel if nd.cols_sel is not None else np.zeros(0, dtype=np.intp))
    # D is not stored: it is C(t, t), regenerated from the generators by the tests
    for name, lst in (("U", U), ("V", V), ("B", B), ("rsel", RS), ("csel", CS)):
        out[f"{prefix}{name}_len"] = np.array([a.size for a in lst], dtype=np.int64)
        out[f"{prefix}{name}"] = np.concatenate(lst) if lst else np.zeros(0)
    out[f"{prefix}meta"] = meta
    out[f"{prefix}r_used"] = np.int64(H.r_used)
    out[f"{prefix}flagged"] = np.int64(H.flagged)


def main():
    hsseig = _import_reference()
    from hsseig import hss, matgen
    from hsseig.backend import kernels as kn
    from hsseig.cauchy import CauchyEvecMatrix
    from hsseig.dc import SolverConfig, adc_solve, update_vectors_hss
    from hsseig.flops import FlopCounter
    from hsseig.secular import RankOneSystem, recompute_weights, solve_secular

    # ---- secular / Loewner / normalizers ------------------------------------
    out = {}
    rng = np.random.default_rng(20251019)
    cases = []
    for k in (1, 2, 3, 17, 150, 600):
        cases.append(("rand%d" % k,) + random_system(rng, k))
    cases.append(("golden",) + (np.array([-1.0, 1.0]), np.array([1.0, 1.0]) / np.sqrt(2.0), 1.0))
    cases.append(("cfg4_1024",) + config4_system(1024, 7))
    names = []
    for name, d, z, rho in cases:
        names.append(name)
        sys_ = RankOneSystem(d, z, rho)
        f = FlopCounter()
        sol = solve_secular(sys_, flops=f)
        lam, gam, mu, iters = kn.secular_all(d, z, rho)
        out[f"{name}_d"], out[f"{name}_z"], out[f"{name}_rho"] = d, z, np.float64(rho)
        out[f"{name}_lam"], out[f"{name}_gamma"], out[f"{name}_mu"] = lam, gam, mu
        out[f"{name}_iters"] = np.int64(iters)
        if d.size >= 2:
            zh = recompute_weights(sys_.d, sol, sys_.z, rho=rho, flops=f)
            C = CauchyEvecMatrix.from_secular(sys_, sol, flops=f)
            out[f"{name}_zhat"], out[f"{name}_v"] = zh, C.v
        out[f"{name}_flops_secular"] = np.int64(f.secular)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "secular.npz"), **out)

    # ---- Cauchy sampling + HSS trees + multiply -----------------------------
    out = {}
    specs = [  # (name, system, leaf, rank_eps, seed)
        ("t256", random_system(np.random.default_rng(11), 256), 64, 1e-16, [0, 3]),
        ("t600", random_system(np.random.default_rng(12), 600), 64, 1e-13, [0, 5]),
        ("c4_2048", config4_system(2048, 3), 128, 1e-13, [0, 0]),
    ]
    for name, (d, z, rho), m, eps, seed in specs:
        sys_ = RankOneSystem(d, z, rho)
        sol = solve_secular(sys_)
        recompute_weights(sys_.d, sol, sys_.z, rho=rho)
        C = CauchyEvecMatrix.from_secular(sys_, sol)
        part = hss.build_partition(C.k, m, C.d, C.gamma, C.mu)
        r = min(hss.estimate_rank(part, C.d, C.gamma, C.mu, eps, 100), part.min_leaf - 10)
        w = r + 10
        Om = np.random.default_rng(seed).standard_normal((C.k, w))
        f = FlopCounter()
        H = hss.rand_hss_construct(C, part, r, p=10, seed=seed, flops=f)
        out[f"{name}_d"], out[f"{name}_z"], out[f"{name}_rho"] = d, z, np.float64(rho)
        out[f"{name}_gamma"], out[f"{name}_mu"] = C.gamma, C.mu
        out[f"{name}_zhat"], out[f"{name}_v"] = C.zhat, C.v
        out[f"{name}_leaf"], out[f"{name}_eps"] = np.int64(m), np.float64(eps)
        out[f"{name}_seed"] = np.array(seed, dtype=np.int64)
        out[f"{name}_ranges"] = np.array(part.ranges, dtype=np.int64)
        out[f"{name}_r"] = np.int64(r)
        out[f"{name}_Y"] = C.multiply(Om)
        out[f"{name}_Z"] = C.transpose_multiply(Om)
        out[f"{name}_flops_construct"] = np.int64(f.hss_construct)
        pack_tree(H, f"{name}_tree_", out)
        X = np.random.default_rng(99).standard_normal((40, C.k))
        f2 = FlopCounter()
        # X = default_rng(99).standard_normal((40, k)) is regenerated by the tests
        out[f"{name}_XH"] = hss.hss_matmul_right(X, H, flops=f2)
        out[f"{name}_flops_mult"] = np.int64(f2.hss_mult)
        # update_vectors_hss on a 48-row Gaussian row block (dc.py:141-171)
        Qold = np.random.default_rng(5).standard_normal((48, C.k))
        f3 = FlopCounter()
        # Qold = default_rng(5).standard_normal((48, k)) is regenerated by the tests
        cfg = SolverConfig(leaf_size=m, hss_threshold=4 * m, rank_eps=eps, oversample=10)
        out[f"{name}_Qnew"] = update_vectors_hss(Qold, C, cfg, seed=seed, flops=f3)
    # rank-starved construction must flag (pkg/tests/test_hss.py:203-208)
    d, z, rho = random_system(np.random.default_rng(13), 256)
    sys_ = RankOneSystem(d, z, rho)
    sol = solve_secular(sys_)
    recompute_weights(sys_.d, sol, sys_.z, rho=rho)
    C = CauchyEvecMatrix.from_secular(sys_, sol)
    part = hss.build_partition(256, 64, C.d, C.gamma, C.mu)
    H = hss.rand_hss_construct(C, part, r=1, p=0, seed=0)
    out["starved_d"], out["starved_z"], out["starved_rho"] = d, z, np.float64(rho)
    out["starved_flagged"] = np.int64(H.flagged)
    out["starved_nflags"] = np.int64(len(H.flags))
    # rank_bound known answer (pkg/tests/test_hss.py:70-72)
    out["rank_bound_2e3_1e-13"] = np.int64(hss.rank_bound(2e3, 1e-13))
    np.savez_compressed(os.path.join(HERE, "hss.npz"), **out)

    # ---- full eigendecompositions -------------------------------------------
    out = {}
    N = 600
    rng = np.random.default_rng(4)
    fams = {
        "toeplitz": matgen.gen_toeplitz(N),
        "kac": matgen.SymTridiagonal(np.zeros(500),
                                     np.sqrt(np.arange(1, 500) * (500 - np.arange(1, 500.0)))),
        "uniform": matgen.SymTridiagonal(rng.uniform(-1, 1, 400), rng.uniform(-1, 1, 399)),
        "cfg5": matgen.SymTridiagonal(rng.uniform(0, 1, 512), rng.uniform(0.5, 1, 511)),
    }
    for name, T in fams.items():
        for method in ("adc-rand", "dense-dc"):
            cfg = SolverConfig(leaf_size=32, hss_threshold=128, rank_eps=1e-13, method=method)
            res = adc_solve(T, cfg)
            tag = f"{name}_{method}"
            out[f"{tag}_lam"] = res.lam
            out[f"{tag}_Qcols"] = res.Q[:, ::8]          # every 8th eigenvector
            out[f"{tag}_orth"] = np.float64(np.abs(res.Q.T @ res.Q - np.eye(T.n)).max() / T.n)
            out[f"{tag}_bwd"] = np.float64(np.abs(T.to_dense() - (res.Q * res.lam) @ res.Q.T).max()
                                           / (T.norm_max() * T.n))
            out[f"{tag}_merges"] = np.array([[m.size, m.kept, m.n_deflated, int(m.used_hss),
                                              m.hss_rank, int(m.fell_back)] for m in res.merges],
                                            dtype=np.int64)
            out[f"{tag}_flops"] = np.array([res.flops.secular, res.flops.update_dense,
                                            res.flops.hss_construct, res.flops.hss_mult],
                                           dtype=np.int64)
        out[f"{name}_a"], out[f"{name}_b"] = T.a, T.b
    np.savez_compressed(os.path.join(HERE, "adc.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
