"""Diagnostics: GPU tree ranks / pivots vs the reference golden trees (run on a GPU box)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from helpers import golden, unpack_tree  # noqa: E402

import paper_1510_04591_b200 as hb  # noqa: E402

g = golden("hss")
for name in ("t256", "t600", "c4_2048"):
    C = hb.CauchyEvecMatrix(g[f"{name}_d"], g[f"{name}_gamma"], g[f"{name}_mu"], g[f"{name}_zhat"], g[f"{name}_v"])
    part = hb.build_partition(C.k, int(g[f"{name}_leaf"]), C.d, C.gamma, C.mu)
    r = int(g[f"{name}_r"])
    H = hb.rand_hss_construct(C, part, r, p=10, seed=[int(s) for s in g[f"{name}_seed"]])
    ref = unpack_tree(g, f"{name}_tree_")
    rU, rV = H.ranks()
    print(name, "w", r + 10)
    for nd, rn in zip(H.nodes, ref):
        if nd.index == H.root:
            continue
        a, b = nd.rows_sel, rn["rsel"]
        n = min(a.size, b.size)
        first = next((i for i in range(n) if a[i] != b[i]), n)
        c, e = nd.cols_sel, rn["csel"]
        m = min(c.size, e.size)
        firstc = next((i for i in range(m) if c[i] != e[i]), m)
        print(f"  node {nd.index:3d} lvl {nd.level} rU {rU[nd.index]:3d}/{rn['rU']:3d} rV {rV[nd.index]:3d}/{rn['rV']:3d}"
              f" first row-pivot diff {first} col {firstc} rres {H._view('rres', __import__('torch').float64, H.ct.n_nodes, 0)[nd.index].item():.2e}")
