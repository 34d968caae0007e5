"""CPU-only checks: C-ABI exports, host-side partition / rank / config logic vs the oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from helpers import config4_system, golden
from oracle import hss_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hsseig_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hsseig_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1510_04591_b200 import _native
    lib = _native.load()            # builds with nvcc if stale; no CUDA call is made
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.EXPORTS, f"{name} missing from the ctypes signature table"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.lib_path()], capture_output=True,
                         text=True, check=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only():
    from paper_1510_04591_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_size_queries_without_gpu():
    from paper_1510_04591_b200 import _native
    lib = _native.load()
    assert lib.hsseig_tree_bytes(32768, 256, 84, 133) > 0
    assert lib.hsseig_sample_work_doubles(32768, 84) >= 2 * 32768 * 84
    assert lib.hsseig_version().startswith(b"hsseig_b200")


@pytest.mark.parametrize("name", ["t256", "t600", "c4_2048"])
def test_partition_and_rank_match_reference(name):
    import paper_1510_04591_b200 as hb
    g = golden("hss")
    k = g[f"{name}_d"].size
    m = int(g[f"{name}_leaf"])
    part = hb.build_partition(k, m, None, None, g[f"{name}_mu"])
    assert [tuple(x) for x in g[f"{name}_ranges"]] == list(part.ranges)
    r = hb.estimate_rank(part, g[f"{name}_d"], g[f"{name}_gamma"], g[f"{name}_mu"],
                         float(g[f"{name}_eps"]))
    assert min(r, part.min_leaf - 10) == int(g[f"{name}_r"])


def test_partition_shift_rule_matches_oracle(rng):
    import paper_1510_04591_b200 as hb
    for _ in range(50):
        k = int(rng.integers(256, 3000))
        m = int(rng.integers(16, 128))
        if k < 2 * m:
            continue
        mu = rng.uniform(1e-3, 1.0, k)
        mu[rng.integers(0, k, k // 10)] = 10.0 ** rng.uniform(-16, -10, k // 10)
        part = hb.build_partition(k, m, None, None, mu)
        assert list(part.ranges) == orc.leaf_ranges(k, m, mu)


def test_partition_rejects_small_order():
    import paper_1510_04591_b200 as hb
    with pytest.raises(ValueError):
        hb.build_partition(100, 64)


def test_rank_bound_known_answer():
    import paper_1510_04591_b200 as hb
    assert hb.rank_bound(2e3, 1e-13) == 33


def test_solver_config_validation():
    import paper_1510_04591_b200 as hb
    with pytest.raises(ValueError):
        hb.SolverConfig(base_size=2)
    with pytest.raises(ValueError):
        hb.SolverConfig(leaf_size=200, hss_threshold=500)
    with pytest.raises(ValueError):
        hb.SolverConfig(method="adc-srrsc-typo")
    cfg = hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
    assert cfg.oversample == 10 and cfg.rank_cap == 100


def test_config_generators():
    import paper_1510_04591_b200 as hb
    d, u, rho = hb.isolated_merge_system(1000, 3)
    d2, u2, _ = config4_system(1000, 3)
    np.testing.assert_array_equal(d, d2)
    np.testing.assert_array_equal(u, u2)
    T = hb.gen_kac(64)
    ev = np.linalg.eigvalsh(T.to_dense())
    np.testing.assert_allclose(ev, -63 + 2 * np.arange(64), atol=1e-11)
    T = hb.gen_toeplitz(50)
    ev = np.linalg.eigvalsh(T.to_dense())
    np.testing.assert_allclose(np.sort(ev), np.sort(2 + 2 * np.cos(np.arange(1, 51) * np.pi / 51)),
                               atol=1e-13)


def test_wave_deflate_matches_oracle_deflation():
    # host side of the level-batched merges (csrc/glue.cu hsseig_wave_deflate / _order)
    # against the oracle's restatement of secular.py:91-156 and dc.py:205-257, merge by merge
    import ctypes
    from oracle import hss_oracle as orc
    from paper_1510_04591_b200 import _native as nat
    lib = nat.load(build_if_missing=False)
    rng = np.random.default_rng(5)
    sizes = [(3, 4), (12, 13), (25, 25), (7, 8), (30, 31)]
    L, Z, bk = [], [], []
    for t, (a, b) in enumerate(sizes):
        l1, l2 = np.sort(rng.uniform(-1, 1, a)), np.sort(rng.uniform(-1, 1, b))
        if t == 1:                      # a near-duplicate pole pair -> Givens rotation
            l2[3] = l1[5] + 1e-17
        z = rng.standard_normal(a + b)
        if t == 2:
            z[4] = 1e-20                # negligible weight -> deflated at its pole
        L.append(np.concatenate([l1, l2]))
        Z.append(z)
        bk.append([0.7, -0.3, 1.1, 0.0, -2.0][t])
    nm = len(sizes)
    n1 = np.array([s[0] for s in sizes], dtype=np.int64)
    n2 = np.array([s[1] for s in sizes], dtype=np.int64)
    nv = n1 + n2
    roff = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
    Lc, Zc, bkc = np.concatenate(L), np.concatenate(Z), np.array(bk)
    nr = int(roff[-1])
    kept, rho_eff = np.empty(nm, dtype=np.int64), np.empty(nm)
    d_out, z_out, src = np.empty(nr), np.empty(nr), np.empty(nr, dtype=np.int64)
    rot_off = np.empty(nm + 1, dtype=np.int64)
    ca, cb, rc, rs = (np.empty(nr, dtype=np.int64), np.empty(nr, dtype=np.int64), np.empty(nr),
                      np.empty(nr))
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    ktot = lib.hsseig_wave_deflate(nm, P(n1), P(n2), P(roff), P(Lc), P(Zc), P(bkc), P(kept),
                                   P(rho_eff), P(d_out), P(z_out), P(src), P(rot_off), P(ca), P(cb),
                                   P(rc), P(rs))
    assert ktot == kept.sum()
    for m in range(nm):
        o, n, a = roff[m], nv[m], n1[m]
        if bk[m] == 0.0:                 # decoupled: sort only
            assert kept[m] == 0 and rot_off[m + 1] == rot_off[m]
            assert np.array_equal(src[o:o + n], np.argsort(L[m], kind="stable"))
            continue
        th = 1.0 if bk[m] >= 0 else -1.0
        z = np.concatenate([Z[m][:a], th * Z[m][a:]]) / np.sqrt(2.0)
        pm = np.argsort(L[m], kind="stable")
        dk, zk, dperm, rots, ldef, nd = orc.deflate(L[m][pm], z[pm], 2.0 * abs(bk[m]))
        k = dk.size
        assert kept[m] == k and rho_eff[m] == 2.0 * abs(bk[m])
        assert np.array_equal(d_out[o:o + k], dk) and np.array_equal(z_out[o:o + k], zk)
        assert np.array_equal(d_out[o + k:o + n], ldef)
        assert np.array_equal(src[o:o + n], pm[dperm])
        pos = np.empty(n, dtype=np.int64)
        pos[pm[dperm]] = np.arange(n)
        r0, r1 = rot_off[m], rot_off[m + 1]
        assert r1 - r0 == len(rots)
        for t, (i, j, c, s) in enumerate(rots):
            assert ca[r0 + t] == pos[pm[i]] and cb[r0 + t] == pos[pm[j]]
            assert rc[r0 + t] == c and rs[r0 + t] == s
    assert kept[1] < nv[1] and kept[2] < nv[2]      # both deflation kinds exercised
    # final order: stable argsort of [roots, deflated poles]
    koff = np.concatenate([[0], np.cumsum(kept)]).astype(np.int64)
    lam = np.concatenate([np.sort(rng.uniform(-3, 3, k)) for k in kept])
    order, lam_out = np.empty(nr, dtype=np.int64), np.empty(nr)
    lib.hsseig_wave_order(nm, P(roff), P(kept), P(koff[:-1].copy()), P(lam), P(d_out), P(order),
                          P(lam_out))
    for m in range(nm):
        o, n, k = roff[m], nv[m], kept[m]
        cat = np.concatenate([lam[koff[m]:koff[m] + k], d_out[o + k:o + n]])
        ref = np.argsort(cat, kind="stable")
        assert np.array_equal(order[o:o + n], ref) and np.array_equal(lam_out[o:o + n], cat[ref])


def test_deflation_tolerance_sums_like_numpy():
    # hsseig_deflate's tol = 8 eps max(max|d|, rho * np.sum(z*z)) (secular.py:91-93) with
    # NumPy's pairwise summation, bit for bit, and a weight placed exactly on the threshold
    # is deflated like the reference does (rho |z_i| <= tol, secular.py:118)
    import ctypes
    from paper_1510_04591_b200 import _native as nat
    lib = nat.load(build_if_missing=False)
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rng = np.random.default_rng(11)
    for n in (1, 5, 8, 9, 127, 128, 129, 1000, 8193, 40000):
        d = np.sort(rng.uniform(-1e-3, 1e-3, n))
        z = rng.standard_normal(n) * np.exp(rng.uniform(-8, 3, n))
        rho = 0.75
        ref = 8.0 * orc.EPS * max(float(np.abs(d).max()), rho * float(np.sum(z * z)))
        out = [np.empty(n), np.empty(n), np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64),
               np.empty(n, dtype=np.int64), np.empty(n), np.empty(n)]
        nrot, tol = ctypes.c_int64(0), ctypes.c_double(0.0)
        lib.hsseig_deflate(P(d), P(z), n, rho, *(P(x) for x in out), ctypes.byref(nrot),
                           ctypes.byref(tol))
        assert tol.value == ref, (n, tol.value, ref)
    # a weight right on the threshold (the tolerance computed the reference's way)
    n = 300
    d = np.linspace(0.0, 1.0, n)
    z = rng.standard_normal(n)
    rho = 1.0
    zz = z * z
    tol = 8.0 * orc.EPS * max(1.0, rho * float(np.sum(zz)))
    z[17] = tol / rho                   # changes the sum only below its last bit
    ref_tol = 8.0 * orc.EPS * max(1.0, rho * float(np.sum(z * z)))
    dk, zk, perm, rots, ldef, nd = orc.deflate(d, z, rho)
    out = [np.empty(n), np.empty(n), np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64),
           np.empty(n, dtype=np.int64), np.empty(n), np.empty(n)]
    nrot, tolo = ctypes.c_int64(0), ctypes.c_double(0.0)
    k = lib.hsseig_deflate(P(d), P(z), n, rho, *(P(x) for x in out), ctypes.byref(nrot),
                           ctypes.byref(tolo))
    assert tolo.value == ref_tol
    assert k == dk.size and np.array_equal(out[2], perm)


def test_recursion_tree_arrays_match_the_recursive_definition():
    """solver._Tree (level-by-level NumPy build) against the recursion of dc.py:194-203 and its
    split modifications (dc.py:82-102), including the merge ids in postorder."""
    import itertools
    from paper_1510_04591_b200 import solver

    def ref_tree(n, base):
        nodes, ids = [], itertools.count()

        def rec(lo, hi, depth):
            if hi - lo <= base:
                nodes.append({"lo": lo, "hi": hi, "depth": depth, "leaf": True})
                return len(nodes) - 1
            m = lo + (hi - lo) // 2
            left = rec(lo, m, depth + 1)
            right = rec(m, hi, depth + 1)
            nodes.append({"lo": lo, "hi": hi, "depth": depth, "leaf": False, "left": left,
                          "right": right, "split": m, "mid": next(ids)})
            return len(nodes) - 1

        return nodes, rec(0, n, 0)

    rng = np.random.default_rng(5)
    for n, base in [(1, 25), (25, 25), (26, 25), (600, 25), (2000, 25), (1023, 3), (4097, 7), (10000, 32)]:
        want, root = ref_tree(n, base)
        got, groot = solver._tree(n, base)
        assert groot == root and len(got) == len(want)
        assert [got[i] for i in range(len(got))] == want
        assert list(got) == want
        for i, nd in enumerate(want):
            if not nd["leaf"]:
                assert i - got.size[i] + 1 == min(j for j in range(i + 1) if want[j]["lo"] == nd["lo"])
        a, b = rng.standard_normal(n), rng.standard_normal(max(n - 1, 0))
        a_ref, _ = solver._plan(a, b, base)
        assert np.array_equal(got.split_diagonal(a, b), a_ref)
        part = a.copy()
        for nd in want:
            if not nd["leaf"] and nd["depth"] < 2:
                part[nd["split"] - 1] -= abs(b[nd["split"] - 1])
                part[nd["split"]] -= abs(b[nd["split"] - 1])
        assert np.array_equal(got.split_diagonal(a, b, 2), part)


def test_tree_flop_counters_equal_the_per_node_definition():
    """hss._construct_flops / hss.mult_flops (sums over node arrays) against the reference's
    per-node accumulation (pkg/src/hsseig/hss.py:251-287, 329-357) on random trees."""
    from paper_1510_04591_b200 import hss
    from paper_1510_04591_b200.flops import cauchy_eval_flops, cpqr_flops, gemm_flops

    class N:
        pass

    def loop_construct(tree, k, w):
        rU, rV = tree.ranks()
        f = 2 * (gemm_flops(k, k, w) + cauchy_eval_flops(k * k))
        for nd in tree.nodes:
            if nd.index == tree.root:
                continue
            if nd.left is None:
                m = nd.hi - nd.lo
                f += cauchy_eval_flops(m * m) + 2 * gemm_flops(m, m, w)
                f += cpqr_flops(w, m, max(int(rU[nd.index]), 1)) + cpqr_flops(w, m, max(int(rV[nd.index]), 1))
            else:
                a, b = nd.left, nd.right
                f += cauchy_eval_flops(int(rU[a] * rV[b]) + int(rU[b] * rV[a]))
                f += 2 * gemm_flops(int(rU[a] + rU[b]), w, max(int(rU[a]), int(rV[b])))
                f += cpqr_flops(w, int(rU[a] + rU[b]), max(int(rU[nd.index]), 1))
                f += cpqr_flops(w, int(rV[a] + rV[b]), max(int(rV[nd.index]), 1))
        rt = tree.nodes[tree.root]
        return f + cauchy_eval_flops(int(rU[rt.left] * rV[rt.right]) + int(rU[rt.right] * rV[rt.left]))

    def loop_mult(tree, P):
        rU, rV = tree.ranks()
        f = 0
        for nd in tree.nodes:
            i = nd.index
            if i == tree.root:
                continue
            m = nd.hi - nd.lo
            if nd.left is None:
                f += gemm_flops(P, m, int(rU[i])) + gemm_flops(P, m, m) + gemm_flops(P, int(rV[i]), m)
            else:
                f += gemm_flops(P, int(rU[nd.left] + rU[nd.right]), int(rU[i]))
                f += gemm_flops(P, int(rV[i]), int(rV[nd.left] + rV[nd.right]))
            f += gemm_flops(P, int(rU[nd.sibling]), int(rV[i]))
        return f

    def loop_srrsc(tree, k):
        rU, rV = tree.ranks()
        f = 0
        for nd in tree.nodes:
            if nd.index == tree.root:
                a, b = nd.left, nd.right
                f += cauchy_eval_flops(int(rU[a] * rV[b]) + int(rU[b] * rV[a]))
                continue
            ncomp = k - (nd.hi - nd.lo)
            if nd.left is None:
                m = nd.hi - nd.lo
                f += cauchy_eval_flops(m * m)
                ps = (m, m)
            else:
                a, b = nd.left, nd.right
                f += cauchy_eval_flops(int(rU[a] * rV[b]) + int(rU[b] * rV[a]))
                ps = (int(rU[a] + rU[b]), int(rV[a] + rV[b]))
            for pc, r in zip(ps, (int(rU[nd.index]), int(rV[nd.index]))):
                f += cauchy_eval_flops((r + 1) * pc * ncomp) + pc * r * r
        return f

    rng = np.random.default_rng(1)
    for nl in [2, 3, 5, 8, 13, 256]:
        nodes = []
        bounds = np.concatenate([[0], np.cumsum(rng.integers(50, 200, nl))])

        def rec(a, b):
            n = N()
            if b - a == 1:
                n.lo, n.hi, n.left, n.right = int(bounds[a]), int(bounds[a + 1]), None, None
            else:
                h = (a + b) // 2
                li, ri = rec(a, h), rec(h, b)
                n.lo, n.hi, n.left, n.right = nodes[li].lo, nodes[ri].hi, li, ri
                nodes[li].sibling, nodes[ri].sibling = ri, li
            n.sibling = None
            n.index = len(nodes)
            nodes.append(n)
            return n.index

        t = N()
        t.root = rec(0, nl)
        t.nodes = nodes
        rU = rng.integers(0, 90, len(nodes)).astype(np.int32)
        rV = rng.integers(0, 90, len(nodes)).astype(np.int32)
        t.ranks = lambda: (rU, rV)
        t._topo = {"leaf": np.array([n.left is None for n in nodes]),
                   "left": np.array([-1 if n.left is None else n.left for n in nodes]),
                   "right": np.array([-1 if n.right is None else n.right for n in nodes]),
                   "sib": np.array([-1 if n.sibling is None else n.sibling for n in nodes]),
                   "m": np.array([n.hi - n.lo for n in nodes])}
        k = int(bounds[-1])
        assert hss._construct_flops(t, k, 88) == loop_construct(t, k, 88)
        assert hss.mult_flops(t, 32768) == loop_mult(t, 32768)
        assert hss._srrsc_flops(t, k) == loop_srrsc(t, k)
