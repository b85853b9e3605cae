"""Bandwidth of repeated reads of an L2-resident vs HBM-resident buffer
(torch sum / copy kernels, CUDA events): is the L2 -> SM path faster than HBM?"""
import torch

for mb in (16, 32, 48, 64, 96, 1024, 4096):
    n = mb * (1 << 20) // 8
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        x.sum()
        y.copy_(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, 2048 // mb)
    e0.record()
    for _ in range(reps):
        x.sum()
    e1.record()
    torch.cuda.synchronize()
    rd = x.numel() * 8 * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(reps):
        y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    cp = 2 * x.numel() * 8 * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(f"{mb:5d} MB: sum read {rd:8.0f} GB/s   copy r+w {cp:8.0f} GB/s")
