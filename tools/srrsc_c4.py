"""ADC1 (SRRSC) construction of the config-4 merge (k = 32768, leaf 128, tol 1e-15): wall ms
per construction, the lazy-search invariant counter, and (argv[2] == "check") the tree
against the full sweep bit for bit.  python tools/srrsc_c4.py [k] [check]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1510_04591_b200 as hb  # noqa: E402
from helpers import config4_system  # noqa: E402

np_ = lambda t: t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d, u, rho = config4_system(k, 0)
s = hb.RankOneSystem(d, u, rho)
sol = hb.solve_secular(s)
hb.recompute_weights(d, sol, u, rho=rho)
C = hb.CauchyEvecMatrix.from_secular(s, sol)
part = hb.build_partition(k, 128, C.d, C.gamma, C.mu)
cap = hb.srrsc_cap(part)
ts = []
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = hb.srrsc_hss_construct(C, part, cap, tol=1e-15, finish=False)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
st = H._status.read()
print(f"k={k} cap={cap} construct ms {['%.2f' % t for t in ts]} invariant={st[7]} max_rank={st[5]}",
      flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "check":
    H = hb.srrsc_hss_construct(C, part, cap, tol=1e-15)
    os.environ["HSSEIG_SRRSC_PRUNE"] = "0"
    F = hb.srrsc_hss_construct(C, part, cap, tol=1e-15)
    same = H.flagged == F.flagged and H.r_used == F.r_used
    for na, nb in zip(H.nodes, F.nodes):
        if na.index == H.root:
            continue
        same &= np.array_equal(na.rows_sel, nb.rows_sel) and np.array_equal(na.cols_sel, nb.cols_sel)
        for x, y in ((na.U, nb.U), (na.V, nb.V), (na.B, nb.B)):
            same &= np.array_equal(np_(x), np_(y))
    print(f"lazy-pruned tree == full sweep: {same} (r_used {H.r_used})", flush=True)
