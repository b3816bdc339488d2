"""Per-launch GEMV time vs. output rows (fixed overhead vs. streaming cost).

  python tools/gemv_scaling.py [family] [d_in]
Graph-replayed launches over L2-exceeding model copies; prints us per launch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "2.06"]
din = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
Ms = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1"])]
kernel = os.environ.get("CCQ_KERNEL", "auto")
s = torch.cuda.Stream()
for dout in (148, 592, 1184, 4096, 14336, 28672, 57344):
    base = random_packed(dout, din, fam, 64, 5)
    one = P.DeviceModel.upload(base)
    copies = max(4, int(300e6 // max(one.payload_bytes, 1)) + 1)
    copies = min(copies, 64)
    ms = [one] + [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 6 + c)) for c in range(copies - 1)]
    for M in Ms:
        x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, dout, device="cuda")

        def body():
            for m in ms:
                P.matmul(m, x, out=y, kernel=kernel, stream=s)
        with torch.cuda.stream(s):
            body()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * len(ms))
        print(f"rows {dout:6d} M {M:3d}: {us:8.2f} us/launch  {one.payload_bytes / us / 1e3:8.1f} GB/s  ({len(ms)} copies)")
    del ms, one
