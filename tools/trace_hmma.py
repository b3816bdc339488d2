"""Per-warp timeline of the tensor-pipe GEMV (gemv_hmma.cu) in a chain of
launches (debug build libccq_b200_trace.so; the trace keeps the last launch).

  python tools/trace_hmma.py [family] [d_in] [d_out] [M] [copies]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), "libccq_b200_trace.so")
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "2.06"]
din = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dout = int(sys.argv[3]) if len(sys.argv) > 3 else 14336
M = int(sys.argv[4]) if len(sys.argv) > 4 else 1
copies = int(sys.argv[5]) if len(sys.argv) > 5 else 12
ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 3 + c)) for c in range(copies)]
x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
y = torch.empty(M, dout, device="cuda")
s = torch.cuda.Stream()


def body():
    for m in ms:
        P.matmul(m, x, out=y, stream=s)


with torch.cuda.stream(s):
    body()
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    body()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(s)
with torch.cuda.stream(s):
    g.replay()
ev1.record(s)
torch.cuda.synchronize()
print(f"chain of {copies}: {ev0.elapsed_time(ev1) * 1000 / copies:.2f} us per launch")
buf = np.zeros(8192 * 8, np.uint64)
assert P.lib().ccq_trace_dump_h(C.c_void_p(buf.ctypes.data), buf.size) == 0
t = buf.reshape(8192, 8).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
base = t[:, 0].min()
names = ["start", "griddep ok", "x max", "x staged", "first stage", "loop end", "exit"]
rel = (t[:, :7] - base) / 1000.0
print("warps", used.sum())
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:12s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
loop = rel[:, 5] - rel[:, 3]
print(f"loop time per warp (staged -> loop end): p50 {np.median(loop):.2f} max {loop.max():.2f} us")
