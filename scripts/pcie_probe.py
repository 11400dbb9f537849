"""PCIe ceiling on this box: pinned host -> device and device -> host copy
rates (torch copies, CUDA events), one direction and both at once."""
import torch
n = 398_131_200
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hm = torch.empty(n // 3, dtype=torch.uint8).pin_memory()
dm = torch.empty(n // 3, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s %.1f" % (5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9))
e0.record()
for _ in range(5):
    hm.copy_(dm, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H GB/s %.1f" % (5 * n / 3 / (e0.elapsed_time(e1) / 1e3) / 1e9))
import time
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        hm.copy_(dm, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("both: H2D %.1f GB/s with D2H %.1f GB/s concurrently" % (5 * n / dt / 1e9, 5 * n / 3 / dt / 1e9))
