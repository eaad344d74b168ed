"""D2H / H2D copy bandwidth with pinned host memory (the e2e leg's copies)."""
import time
import torch
n = 34799616 // 8
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
for direction in ("d2h", "h2d"):
    for _ in range(3):
        (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(f"{direction}: {n * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.3f} ms per 34.8 MB)")
