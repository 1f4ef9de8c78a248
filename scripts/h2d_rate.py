"""Host<->device copy rates on the box: the C5 per-object input (439 MB H2D) alone and with the
result read-back (128 MB D2H) running concurrently; the bound of bench.py's e2e figure."""
import torch, time
n = 439_082_496
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D {n/1e6:.0f} MB: {ms:.2f} ms = {n/ms/1e6:.1f} GB/s")
# D2H concurrently
h2 = torch.empty(128_000_016, dtype=torch.uint8).pin_memory()
d2 = torch.empty(128_000_016, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"H2D 439 MB + D2H 128 MB concurrently: {e0.elapsed_time(e1):.2f} ms")
