"""Where does the GPU HSS construction differ from the reference's?  For one merge system,
the reference algorithm (oracle restatement, pinned to the reference) is run with one GPU
piece swapped in at a time: the interpolative decomposition, the sample Y/Z, the Cauchy
blocks; then the GPU construction itself.  Reports tree ranks vs the oracle's, the HSS
error max|H - C| and orthogonality.

    python tools/orth_bisect.py kac            # Kac N=8000 top merge (tools/kac8000_top.npz)
    python tools/orth_bisect.py c4 8192        # BASELINE config-4 system, leaf 128
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1510_04591_b200 as hb  # noqa: E402
from oracle import hss_oracle as orc  # noqa: E402
from paper_1510_04591_b200 import hss as hhss  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "kac"
if mode == "kac":
    z = np.load("tools/kac8000_top.npz")
    G = orc.Generators(z["d"], z["gamma"], z["mu"], z["zhat"], z["v"])
    leaf, seed = 200, [int(s) for s in z["seed"]]
else:
    n = int(sys.argv[2])
    d, u, rho = hb.isolated_merge_system(n, 0)
    G, _, _ = orc.generators_from_roots(d, u, rho)
    leaf, seed = 128, [0, 0]
k = G.k
dense_ok = k <= orc.DENSE_LIMIT * 4
orc.DENSE_LIMIT = max(orc.DENSE_LIMIT, k)
Cref = hb.CauchyEvecMatrix(G.d, G.gam, G.mu, G.zh, G.v)
ranges = orc.leaf_ranges(k, leaf, G.mu)
r = min(orc.rank_estimate(ranges, G.d, G.gam, G.mu, 1e-13), min(h - l for l, h in ranges) - 10)
w = r + 10
Om = orc.sample_block(k, w, seed)
Cd = Cref.to_dense()
I = torch.eye(k, dtype=torch.float64, device="cuda")
print(f"{mode}: k={k} leaf={leaf} r={r} w={w} leaves={len(ranges)}")
base = {}


def ranks_of(T):
    ru = np.array([nd.U.shape[1] if nd.U is not None else -1 for nd in T.nodes])
    rv = np.array([nd.V.shape[1] if nd.V is not None else -1 for nd in T.nodes])
    return ru[:-1], rv[:-1]


def report(label, T=None, Hd=None, ranks=None):
    if Hd is None:
        Hd = torch.as_tensor(orc.hss_apply_right(np.eye(k), T), device="cuda")
    o = float((Hd.T @ Hd - I).abs().max())
    e = float((Hd - Cd).abs().max())
    ru, rv = ranks_of(T) if ranks is None else ranks
    if not base:
        base.update(ru=ru, rv=rv)
    du, dv = ru - base["ru"], rv - base["rv"]
    print(f"{label:30s} orth {o:.3e}  max|H-C| {e:.3e}  dU mean {du.mean():+.2f} [{du.min():+d},"
          f"{du.max():+d}]  dV mean {dv.mean():+.2f} [{dv.min():+d},{dv.max():+d}]  "
          f"sum rU {ru.sum()} rV {rv.sum()}", flush=True)


report("A oracle (reference algo)", orc.rand_construct(G, ranges, r, 10, seed))
orig_id = orc.row_id


def gpu_id(M, tol, max_rank):
    X, J, res, sat = hhss._interp_rows(torch.as_tensor(M, device="cuda"), tol, max_rank)
    return X.cpu().numpy(), J, res, sat


Yg, Zg = Cref.sample(torch.as_tensor(Om, device="cuda"))
Yg, Zg = Yg.cpu().numpy(), Zg.cpu().numpy()
Yn, Zn = G.times(Om), G.t_times(Om)
print(f"sample diff vs numpy: Y {np.abs(Yg - Yn).max():.3e} (|Y| {np.abs(Yn).max():.2e})  "
      f"Z {np.abs(Zg - Zn).max():.3e}")


class GY(orc.Generators):
    def times(self, X, flops=None, block=512):
        return Yg.copy()

    def t_times(self, X, flops=None, block=512):
        return Zg.copy()


class GB(orc.Generators):
    def block(self, rows, cols, flops=None, phase="hss_construct"):
        return Cref.block(np.asarray(rows), np.asarray(cols)).cpu().numpy()

    def times(self, X, flops=None, block=512):
        return Yn.copy()

    def t_times(self, X, flops=None, block=512):
        return Zn.copy()


class GYB(GB):
    def times(self, X, flops=None, block=512):
        return Yg.copy()

    def t_times(self, X, flops=None, block=512):
        return Zg.copy()


args = (G.d, G.gam, G.mu, G.zh, G.v)
orc.row_id = gpu_id
report("B oracle + GPU ID", orc.rand_construct(G, ranges, r, 10, seed))
orc.row_id = orig_id
report("C oracle + GPU Y/Z", orc.rand_construct(GY(*args), ranges, r, 10, seed))
report("D oracle + GPU blocks (D, B)", orc.rand_construct(GB(*args), ranges, r, 10, seed))
orc.row_id = gpu_id
report("F oracle + GPU ID, Y/Z, blocks", orc.rand_construct(GYB(*args), ranges, r, 10, seed))
orc.row_id = orig_id
part = hb.build_partition(k, leaf, Cref.d, Cref.gamma, Cref.mu)
H = hb.rand_hss_construct(Cref, part, r, p=10, seed=seed)
rU, rV = H.ranks()
report("G GPU construction", Hd=hb.hss_matmul_right(I, H), ranks=(rU[:-1], rV[:-1]))
