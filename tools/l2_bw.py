"""Measure read bandwidth of an L2-resident buffer vs an HBM-sized buffer (torch sum)."""
import torch

def bw(nbytes, reps):
    x = torch.ones(nbytes // 8, dtype=torch.float64, device="cuda")
    for _ in range(3):
        x.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        x.sum()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9

for mb in (16, 32, 64, 96, 4096):
    print(f"{mb:5d} MB: {bw(mb << 20, 200 if mb < 1000 else 10):8.0f} GB/s")
