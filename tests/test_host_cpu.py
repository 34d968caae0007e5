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
