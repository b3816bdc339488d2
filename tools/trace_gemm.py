"""Per-decode-warp cycle breakdown of the tcgen05 GEMM (debug build)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), "libccq_b200_trace.so")
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
din, dout = 4096, 14336
m = P.DeviceModel.upload(random_packed(dout, din, 2, 64, 3))
x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
y = torch.empty(M, dout, device="cuda")
for _ in range(3):
    P.matmul(m, x, out=y, kernel="gemm")
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
assert P.lib().ccq_gemm_trace_dump(C.c_void_p(buf.ctypes.data), buf.size) == 0
raw = buf.reshape(-1, 8).astype(np.float64)
mm = raw[raw[:, 7] > 0][:, 5:8]
print(f"MMA warp: wait A p50 {np.median(mm[:, 0]):.0f}  wait B p50 {np.median(mm[:, 1]):.0f}  total p50 {np.median(mm[:, 2]):.0f} cycles")
t = raw[:, :5]
t = t[t[:, 4] > 0]
names = ["wait code", "decode", "wait empty", "st+wait+arrive", "total"]
for i, n in enumerate(names):
    print(f"{n:16s} p50 {np.median(t[:, i]):9.0f} cycles  ({100 * np.median(t[:, i] / t[:, 4]):5.1f}%)")
