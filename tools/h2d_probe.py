"""Pinned host->device copy bandwidth (the e2e ceiling): 112 MB like C2's X."""
import torch, time
x = torch.empty(28_000_000, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("h2d 112MB ms", min(ts), "GB/s", 112e6 / (min(ts) / 1e3) / 1e9)
# two halves on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h = x.numel() // 2
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d[:h].copy_(x[:h], non_blocking=True)
    with torch.cuda.stream(s2): d[h:].copy_(x[h:], non_blocking=True)
    torch.cuda.synchronize()
print("2-stream GB/s", 112e6 * 10 / (time.perf_counter() - t) / 1e9)
