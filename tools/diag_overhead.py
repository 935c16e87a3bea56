"""Diagnose host/launch overheads around predict and predict_host (GPU box)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_12491_b200 as B
from synth import make_config, gen_x_torch, gen_x

c, m = make_config("C2")
X = gen_x_torch(2, 0, c.n_rows, 28, device="cuda")
g = B.Model(m)
out = torch.empty(c.n_rows, dtype=torch.int32, device="cuda")
for _ in range(3): g.predict(X, out=out)
torch.cuda.synchronize()
# host enqueue cost
t = time.perf_counter()
for _ in range(20): g.predict(X, out=out)
t_enq = (time.perf_counter() - t) / 20
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): g.predict(X, out=out)
torch.cuda.synchronize()
t_back = (time.perf_counter() - t) / 20
B.hot_kernel_timing(True); B.hot_kernel_time()
for _ in range(20): g.predict(X, out=out)
torch.cuda.synchronize()
hot, n = B.hot_kernel_time(); B.hot_kernel_timing(False)
print(f"host enqueue/predict {t_enq*1e6:.1f} us, back-to-back {t_back*1e3:.3f} ms, hot kernel {hot/n:.3f} ms")
# H2D bandwidth
Xh = torch.from_numpy(gen_x(2, 0, c.n_rows, 28)).pin_memory()
Xd = torch.empty_like(Xh, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): Xd.copy_(Xh, non_blocking=True)
torch.cuda.synchronize(); t_h2d = (time.perf_counter() - t) / 5
print(f"H2D 112MB pinned: {t_h2d*1e3:.2f} ms = {112e6/t_h2d/1e9:.1f} GB/s")
oh = torch.empty(c.n_rows, dtype=torch.int32).pin_memory()
for i in range(4):
    t = time.perf_counter(); g.predict_host(Xh, out=oh); print(f"predict_host {(time.perf_counter()-t)*1e3:.2f} ms")
print(B.Model(make_config("C2")[1]).info(), len(g._keep.arrs))
