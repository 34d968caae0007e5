"""Finer host timing of one solve_subtree level loop (statement anchors), config 5 by default."""
import collections
import inspect
import sys
import time

sys.path.insert(0, ".")
import paper_1510_04591_b200.solver as S  # noqa: E402

marks = [
    ("zrow = src_rows[np.repeat", "A_zrows_wait"),
    ("ktot = int(lib.hsseig_wave_deflate", "B_z_assembly"),
    ("wd = np.empty(nm, dtype=np.int64)", "C_deflate"),
    ("segs = np.flatnonzero(kept > 0)", "D_compact"),
    ("nvs = nv[segs]", "E_kidx"),
    ("st0 = np.zeros((nseg, 8), dtype=np.int64)", "F_tiles"),
    ("W = torch.empty(max(int(woff[-1]), 2), **f64)", "G_pack_send"),
    ("roots_ready.synchronize()", "H_enqueue"),
    ("bad_b = (stv[:, 1] < ks)", "I_sync2"),
    ("order = np.empty(nrows, dtype=np.int64)", "J_hss_lam"),
    ("A = torch.empty(int(ooff[-1]), **f64)", "K_order"),
    ("sel = np.flatnonzero(has_parent[ms])", "L_desc"),
    ("nat.check(lib.hsseig_wave_gather(", "M_rows_pack"),
    ("for q, m in enumerate(segs.tolist()):", "N_gather_enqueue"),
]
src = inspect.getsource(S.solve_subtree)
out = []
for ln in src.split("\n"):
    st = ln.strip()
    for key, name in marks:
        if st.startswith(key):
            ind = ln[:len(ln) - len(ln.lstrip())]
            out.append(f"{ind}_T['{name}'] += time.perf_counter() - _t0; _t0 = time.perf_counter()")
    if st.startswith("for depth in range("):
        out.append(ln)
        ind = ln[:len(ln) - len(ln.lstrip())] + "    "
        out.append(f"{ind}_t0 = time.perf_counter()")
        continue
    if st.startswith("# boundary rows of the children (sync 1"):
        ind = ln[:len(ln) - len(ln.lstrip())]
        out.append(f"{ind}_T['O_records_setup'] += time.perf_counter() - _t0; _t0 = time.perf_counter()")
    out.append(ln)
ns = dict(S.__dict__)
ns["time"] = time
_T = collections.Counter()
ns["_T"] = _T
exec("\n".join(out), ns)
S.solve_subtree = ns["solve_subtree"]
import torch  # noqa: E402

import paper_1510_04591_b200 as hb  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
T = hb.gen_config5(n, 0)
cfg = hb.SolverConfig(rank_eps=1e-13)
hb.adc_solve(T, cfg)
torch.cuda.synchronize()
_T.clear()
t0 = time.perf_counter()
hb.adc_solve(T, cfg)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
for k in sorted(_T):
    print(f"{k:20s} {1e3 * _T[k]:8.2f} ms")
