# instrument solve_subtree with section timers (monkeypatch by source transformation)
import sys, time, re, os
sys.path.insert(0, ".")
import paper_1510_04591_b200.solver as S
import inspect, textwrap, collections
src = inspect.getsource(S.solve_subtree)
marks = [
 ("src_rows = rows_h", "setup"),
 ("bk = np.ascontiguousarray(b[sp_m - 1], dtype=np.float64)", "zrows_sync"),
 ("wd = np.empty(nm, dtype=np.int64)", "deflate"),
 ("W = torch.empty(max(int(woff[-1]), 2), **f64)", "index_pack"),
 ("roots_ready.synchronize()", "enqueue_gpu"),
 ("bad_b = (stv[:, 1] < ks) | ((ks >= 2) & (stv[:, 2] < ks))", "sync2"),
 ("order = np.empty(nrows, dtype=np.int64)", "hss_and_lam"),
 ("del W, Qk", "order_gather"),
]
lines = src.split("\n")
out = []
for ln in lines:
    stripped = ln.strip()
    for key, name in marks:
        if stripped.startswith(key):
            ind = ln[:len(ln) - len(ln.lstrip())]
            out.append(f"{ind}_T['{name}'] += time.perf_counter() - _t0; _t0 = time.perf_counter()")
    out.append(ln)
    if stripped.startswith("for depth in range("):
        ind = ln[:len(ln) - len(ln.lstrip())] + "    "
        out.append(f"{ind}_t0 = time.perf_counter()")
src2 = "\n".join(out)
# end of loop body marker: before 'n = int(hi_a[-1] - lo_a[-1])'
src2 = src2.replace("    n = int(hi_a[-1] - lo_a[-1])", "    n = int(hi_a[-1] - lo_a[-1])", 1)
ns = dict(S.__dict__)
ns["time"] = time
_T = collections.Counter()
ns["_T"] = _T
exec(src2, ns)
S.solve_subtree = ns["solve_subtree"]
import paper_1510_04591_b200 as hb, torch
cfg_id, n = sys.argv[1], int(sys.argv[2])
T = hb.gen_config5(n, 0) if cfg_id == "5" else hb.gen_uniform(n, 0)
cfg = hb.SolverConfig(rank_eps=1e-13) if cfg_id == "5" else hb.SolverConfig(leaf_size=64, hss_threshold=256, rank_eps=1e-13)
hb.adc_solve(T, cfg); torch.cuda.synchronize()
_T.clear()
t0 = time.perf_counter(); hb.adc_solve(T, cfg); torch.cuda.synchronize(); w = time.perf_counter() - t0
print("wall", w)
for k, v in _T.most_common(): print(f"{k:14s} {1e3*v:8.2f} ms")
