"""Where a small predict's time goes (C1: one depth-3 tree, 150 rows): host
microseconds per call of the Python binding, the bare C call, and pieces."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_12491_b200 as B  # noqa: E402
from synth import iris_like_x, make_config  # noqa: E402


def per_call(f, n=3000):
    for _ in range(100):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


cfg, m = make_config("C1")
X = torch.from_numpy(iris_like_x(1)).cuda()
g = B.Model(m)
out = torch.empty(150, dtype=torch.int32, device="cuda")
lib = B.lib()
xp, op, sp = X.data_ptr(), out.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)
print("predict (binding) us/call", per_call(lambda: g.predict(X, out=out)))
print("bare C call us/call", per_call(lambda: lib.bridger_predict(g._h, xp, 150, 4, op, sp)))
print("current_stream us", per_call(lambda: torch.cuda.current_stream(X.device)))
print("_x us", per_call(lambda: g._x(X)))
print("data_ptr x2 us", per_call(lambda: (X.data_ptr(), out.data_ptr())))
print("n_rows=0 C call us", per_call(lambda: lib.bridger_predict(g._h, xp, 0, 4, op, sp)))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(300):
    ev[0].record()
    lib.bridger_predict(g._h, xp, 150, 4, op, sp)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
print("bare C call, event us median", float(np.median(ts)))

# the same predict captured once into a CUDA graph (serving path)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    g.predict(X, out=out)
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    g.predict(X, out=out)
print("graph replay us/call", per_call(graph.replay))
ts = []
for _ in range(300):
    ev[0].record()
    graph.replay()
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
print("graph replay, event us median", float(np.median(ts)))
