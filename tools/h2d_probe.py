import torch, time
n = 238464000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D {n/ms/1e6:.1f} GB/s ({ms:.2f} ms per 238 MB)")
# two streams concurrently (halves)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
torch.cuda.synchronize(); e0.record()
for _ in range(10):
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
print("2 streams", n / (e0.elapsed_time(e1) / 10) / 1e6, "GB/s")
