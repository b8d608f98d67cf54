"""Dev: pinned PCIe copy throughput on the box (D2H 512 MB, with a concurrent 64 MB H2D): the e2e ceiling."""
import torch, time
n = 512 * 1024 * 1024
d = torch.empty(n, dtype=torch.uint8, device='cuda')
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(64*1024*1024, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(64*1024*1024, dtype=torch.uint8, device='cuda')
for _ in range(2): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
for rep in range(5):
    t=time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"D2H 512MB: {n/dt/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
for rep in range(3):
    t=time.perf_counter()
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"D2H 512MB + concurrent H2D 64MB: {n/dt/1e9:.1f} GB/s (D2H)")
