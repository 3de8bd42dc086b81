"""PCIe copy bandwidth on the box: H2D, D2H alone and concurrently (pinned)."""
import time
import torch
n = 1 << 29  # 4 GiB of float64
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t
for _ in range(2):
    run(True, True)
for name, a, b in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
    t = min(run(a, b) for _ in range(3))
    print(f"{name}: {t*1e3:.1f} ms, {8*n*(a+b)/t/1e9:.1f} GB/s total", flush=True)
print(torch.cuda.get_device_properties(0))
