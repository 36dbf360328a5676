"""Raw pinned-host -> device and device -> host copy bandwidth (the e2e leg's bound), one and two streams."""
import torch

n = 1428462752 // 2  # bench.py's per-step H2D bytes, as bf16
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"H2D one stream: {n * 2 / ms / 1e6:.1f} GB/s ({ms:.2f} ms for {n * 2 / 1e9:.2f} GB)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"H2D two streams: {n * 2 / ms / 1e6:.1f} GB/s")
e0.record()
for _ in range(5):
    h.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"D2H one stream: {n * 2 / ms / 1e6:.1f} GB/s")
