"""Graph-timed tcgen05 GEMM at small/medium M on the configs[1] shapes (all families)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402

if os.environ.get("CCQ_LIB"):  # experiment builds (tools only)
    P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ["CCQ_LIB"])
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

s = torch.cuda.Stream()
for fname in sys.argv[1].split(",") if len(sys.argv) > 1 else ["2.06"]:
    for din, dout in ((4096, 14336), (14336, 4096)):
        copies = max(2, int(160e6 // (din * dout * 0.3)) + 1)
        ms = [P.DeviceModel.upload(random_packed(dout, din, P.FAMILIES[fname], 64, 3 + c)) for c in range(copies)]
        for M in (16, 32, 64, 128, 256):
            x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
            y = torch.empty(M, dout, device="cuda")

            def body():
                for m in ms:
                    P.matmul(m, x, out=y, stream=s, kernel="gemm")
            with torch.cuda.stream(s):
                body()
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(5):
                    g.replay()
                e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * copies)
            print(f"{fname} {din}x{dout} M={M:4d}: {us:8.2f} us  {2 * M * din * dout / us / 1e6:7.1f} TFLOP/s")
        del ms
