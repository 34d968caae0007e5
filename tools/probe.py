"""Box probe: host cores/RAM, cuBLAS DGEMM FP64 rate, QR timing (setup cost for config 4)."""
import os, time, subprocess
import torch
print("cpus", os.cpu_count(), "sched", len(os.sched_getaffinity(0)))
print(subprocess.run("free -g; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv", shell=True, capture_output=True, text=True).stdout)
dev = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"DGEMM {n}: {2*n**3/ms/1e9:.2f} TF/s")
for n in (8192, 16384):
    g = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(); t = time.time()
    q, _ = torch.linalg.qr(g)
    torch.cuda.synchronize(); print(f"QR {n}: {time.time()-t:.2f}s")
    del g, q
