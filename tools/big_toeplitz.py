import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1510_04591_b200 as hb
n = 65536
T = hb.gen_toeplitz(n)
cfg = hb.SolverConfig(rank_eps=1e-13)
t0 = time.perf_counter()
res = hb.adc_solve(T, cfg)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
closed = np.sort(2 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
print("wall", dt, "merges", len(res.merges), "hss", sum(m.used_hss for m in res.merges),
      "top kept", res.merges[-1].kept, "eig err", np.abs(res.lam - closed).max(),
      "peak GB", torch.cuda.max_memory_allocated() / 1e9)
cols = torch.arange(0, n, 257, device="cuda")
G = res.Q[:, cols].T @ res.Q
G[torch.arange(cols.numel(), device="cuda"), cols] -= 1
print("orth (sampled cols)", float(G.abs().max()) / n)
for m in res.merges:
    if m.size >= 4096:
        print(m.size, m.kept, m.used_hss, m.fell_back, m.hss_rank)
t0 = time.perf_counter()
res = hb.adc_solve(T, cfg)
torch.cuda.synchronize()
print("second run wall", time.perf_counter() - t0)
