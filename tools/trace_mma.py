"""Per-warp timeline of the tensor-pipe GEMV (debug build libccq_b200_trace.so).

  python tools/trace_mma.py [family] [d_in] [d_out] [M]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ.get("CCQ_TRACE_LIB", "libccq_b200_trace.so"))
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "2.06"]
din = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dout = int(sys.argv[3]) if len(sys.argv) > 3 else 14336
M = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 3 + c)) for c in range(6)]
x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
y = torch.empty(M, dout, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for r in range(3):
        for m in ms:
            P.matmul(m, x, out=y, stream=s)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
assert P.lib().ccq_trace_dump_mma(C.c_void_p(buf.ctypes.data), buf.size) == 0
t = buf.reshape(4096, 8).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
base = t[:, 0].min()
names = ["start", "griddep ok", "x max done", "x staged", "first data", "loop end", "exit"]
rel = (t[:, :7] - base) / 1000.0
print("warps", used.sum(), "items/warp min", t[:, 7].min(), "max", t[:, 7].max(), "mean", t[:, 7].mean())
for i, n in enumerate(names):
    col = rel[:, i]
    col = col[t[:, i] > 0]
    if col.size:
        print(f"{n:11s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
act = (t[:, 4] > 0) & (t[:, 5] > 0)
loop = (t[act, 5] - t[act, 4]) / 1000.0
print(f"loop per warp p50 {np.median(loop):.2f} max {loop.max():.2f} us; per item p50 {np.median(loop / np.maximum(t[act, 7], 1)):.3f} us")
