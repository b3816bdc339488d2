"""Stream-K GEMM timeline per CTA (trace build of the stream-K experiment:
apply tools/experiments/gemm_streamk.patch first - the adopted kernel has no
ccq_gemm_sktrace_dump): start, first stage, segment ends (MMA commits),
epilogue phases, CTA end (profiles/r02_gemm_streamk.txt).

  python tools/trace_sk.py FAM D_IN D_OUT M
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

fam, din, dout, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
m = P.DeviceModel.upload(random_packed(dout, din, P.FAMILIES[fam], 64, 3))
x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
y = torch.empty(M, dout, device="cuda")
for _ in range(3):
    P.matmul(m, x, out=y, kernel="gemm")
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
P.matmul(m, x, out=y, kernel="gemm")
ev1.record()
torch.cuda.synchronize()
print(f"one call {ev0.elapsed_time(ev1) * 1000:.1f} us (includes prepass)")
buf = (C.c_ulonglong * (1024 * 16))()
assert P.lib().ccq_gemm_sktrace_dump(buf, 1024 * 16) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
base = t[:, 0].min()
rel = np.where(t > 0, (t - base) / 1000.0, np.nan)
names = ["start", "seg0 first stage", "seg0 mma done", "seg0 epi done", "seg1 acc free", "seg1 mma done",
         "seg1 epi done", "end", "e0 tmem_full", "e0 griddep", "e0 flags", "e0 loop done", "e1 tmem_full",
         "e1 griddep", "e1 flags", "e1 loop done"]
print("CTAs", t.shape[0])
for i, n in enumerate(names):
    c = rel[:, i]
    c = c[~np.isnan(c)]
    if len(c):
        print(f"{n:18s} n {len(c):4d} min {c.min():7.2f} p50 {np.median(c):7.2f} p90 {np.percentile(c, 90):7.2f} max {c.max():7.2f}")



# per-CTA view (stream-K segment kinds recomputed host-side)
G = 1 if M > 128 else (2 if M > 64 else 4)
spt = (din // 64 + G - 1) // G
ntl = (M + (256 if M > 192 else 64) - 1) // (256 if M > 192 else 64)
T = ((dout + 127) // 128) * ntl * spt
Pn = t.shape[0]
print("cta: [seg kinds] mma0 tf0 gd0 fl0 lp0 epi0 acc1 mma1 tf1 gd1 fl1 lp1 epi1 end (us)")
for b in list(range(0, 12)) + list(range(Pn - 4, Pn)):
    lo, hi = b * T // Pn, (b + 1) * T // Pn
    tA = lo // spt
    endA = (tA + 1) * spt
    kinds = ["1"] if hi < endA else (["0" if lo == tA * spt else "2"] if hi == endA else ["1(head)", "0" if lo == tA * spt else "2"])
    print(b, kinds, lo, hi, " ".join(f"{v:6.2f}" for v in rel[b, [2, 8, 9, 10, 11, 3, 4, 5, 12, 13, 14, 15, 6, 7]]))
