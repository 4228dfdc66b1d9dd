"""Achievable HBM read bandwidth on this GPU (diagnostic): a read-only
reduction over 8 GiB, CUDA events, best of 10.  MEASURED_PEAKS.json's
hbm_gbs is a copy (read + write); a weight stream is read-only."""
import torch

x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda").view(torch.int64)
x.fill_(1)
best = 1e9
for _ in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    torch.amax(x)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"read-only amax over 8 GiB: {8 * 2**30 / best / 1e6:.0f} GB/s")
