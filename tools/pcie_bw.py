"""Pinned host<->device bandwidth on this box: H2D, D2H and both directions at once."""
import torch

n = 1 << 29   # 4 GiB of float64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 8 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H {gb / t * 1e3:.1f} GB/s")
t = timed(both)
print(f"bidirectional {2 * gb / t * 1e3:.1f} GB/s total ({t:.1f} ms for {gb:.1f} GB each way)")
