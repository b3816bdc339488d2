"""Time the tcgen05 GEMM on BASELINE configs[4] (8192 -> 28672, M = 4096) per family / out dtype."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fams = sys.argv[1].split(",") if len(sys.argv) > 1 else ["2.06", "2.5", "2.75"]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
for fname in fams:
    m = P.DeviceModel.upload(random_packed(28672, 8192, P.FAMILIES[fname], 64, 5))
    x = torch.randn(M, 8192, device="cuda").to(torch.bfloat16)
    for od in (torch.float32, torch.bfloat16):
        y = torch.empty(M, 28672, device="cuda", dtype=od)
        for _ in range(2):
            P.matmul(m, x, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.matmul(m, x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{fname} M={M} out={od}: {ms:.3f} ms  {2 * M * 8192 * 28672 / ms / 1e9:.1f} TFLOP/s")
