"""Measure the dense int8 tensor peak on this B200 (cuBLASLt s8 x s8 -> s32 via
torch._int_mm, 8192^3, best of 10 and sustained 3 s), the roofline denominator
for the path-contraction kernel K2.  Writes profiles/int8_peak.json."""
import json
import os
import time

import torch

n = 8192
a = torch.randint(-2, 2, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-2, 2, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
burst = 2 * n ** 3 / best / 1e12
t0 = time.time()
it = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 3.0:
    torch._int_mm(a, b)
    it += 1
e1.record()
torch.cuda.synchronize()
sustained = 2 * n ** 3 * it / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"int8_tops_burst": burst, "int8_tops_sustained": sustained, "how": "torch._int_mm (cuBLASLt) 8192^3 s8xs8->s32, best of 10 / back-to-back 3 s",
       "gpu": torch.cuda.get_device_name()}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/int8_peak.json", "w"), indent=1)
print(out)
