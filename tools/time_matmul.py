"""Time ccq matmul (GEMV or tcgen05 GEMM) per (family, d_in, d_out, M):
CUDA events around graph-captured launches, rotating over weight copies so
the working set exceeds L2.  Not the driver bench; a tuning tool."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402

if os.environ.get("CCQ_LIB"):  # experiment builds (tools only)
    P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ["CCQ_LIB"])
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="2.06")
ap.add_argument("--shapes", default="4096x14336")  # d_in x d_out
ap.add_argument("--M", default="1,4,16,32,64,128,256")
ap.add_argument("--kernel", default="auto")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
fam = P.FAMILIES[a.family]
peak_bw = 6546.6
for shp in a.shapes.split(","):
    din, dout = map(int, shp.split("x"))
    copies = max(2, int(200e6 // (din * dout * 0.3)) + 1)
    ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 11 + c)) for c in range(copies)]
    pb = ms[0].payload_bytes
    for M in map(int, a.M.split(",")):
        x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, dout, device="cuda")
        s = torch.cuda.Stream()
        def body():
            for m in ms:
                P.matmul(m, x, out=y, kernel=a.kernel, stream=s)
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
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(a.reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (a.reps * copies)
        print(json.dumps({"family": a.family, "kernel": a.kernel, "d_in": din, "d_out": dout, "M": M, "us": round(us, 2),
                          "packed_GBps": round(pb / us / 1e3, 1), "hbm_frac": round(pb / us / 1e3 / peak_bw, 3),
                          "TFLOPs": round(2 * M * din * dout / us / 1e6, 1)}))
        del g
    del ms
