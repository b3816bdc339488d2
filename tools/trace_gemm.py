"""Per-decode-warp cycle breakdown of the tcgen05 GEMM (debug build).

usage: trace_gemm.py [M,...] [exp,...]   exp: 0 normal, 1 skip decode math,
2 skip MMAs, 3 skip TMEM stores (results meaningless for 1-3)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), "libccq_b200_trace.so")
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

Ms = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16").split(",")]
exps = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
fam = os.environ.get("FAM", "2.06")
din, dout = int(os.environ.get("DIN", "4096")), int(os.environ.get("DOUT", "14336"))
m = P.DeviceModel.upload(random_packed(dout, din, P.FAMILIES[fam], 64, 3))
for M in Ms:
    x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, dout, device="cuda")
    for ex in exps:
        assert P.lib().ccq_gemm_trace_exp(ex) == 0
        for _ in range(3):
            P.matmul(m, x, out=y, kernel="gemm")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            P.matmul(m, x, out=y, kernel="gemm")
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        buf = np.zeros(4096 * 8, np.uint64)
        assert P.lib().ccq_gemm_trace_dump(C.c_void_p(buf.ctypes.data), buf.size) == 0
        raw = buf.reshape(-1, 8).astype(np.float64)
        print(f"== {fam} M={M} exp={ex}: {us:.2f} us per launch (L2-warm, eager)")
        mm = raw[raw[:, 7] > 0][:, 5:8]
        print(f"MMA warp: wait full p50 {np.median(mm[:, 0]):.0f}  in-issue p50 {np.median(mm[:, 1]):.0f}"
              f"  total p50 {np.median(mm[:, 2]):.0f} cycles")
        t = raw[:, :5]
        t = t[t[:, 4] > 0]
        names = ["wait code", "decode", "wait empty", "st+wait+arrive", "total"]
        b2 = np.zeros(4096 * 4, np.uint64)
        assert P.lib().ccq_gemm_trace_dump2(C.c_void_p(b2.ctypes.data), b2.size) == 0
        r2 = b2.reshape(-1, 4).astype(np.float64)
        live = r2[raw.reshape(-1, 8)[: r2.shape[0], 4] > 0] if False else r2[r2[:, 0] > 0]
        prod = r2[::12][:, 3]
        print(f"code ring: first arrival p50 {np.median(live[:, 0]):.0f}  waits>1000cyc p50 {np.median(live[:, 1]):.0f}"
              f"  max wait p50 {np.median(live[:, 2]):.0f}  producer wait-empty p50 {np.median(prod[prod > 0]) if (prod > 0).any() else 0:.0f}")
        for i, n in enumerate(names):
            print(f"{n:16s} p50 {np.median(t[:, i]):9.0f} cycles  ({100 * np.median(t[:, i] / t[:, 4]):5.1f}%)")
