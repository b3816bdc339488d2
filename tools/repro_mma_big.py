"""Repro: tensor-pipe GEMV on 8192 -> 28672 (configs[4] shape) at M = 5..8."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[os.environ.get("FAM", "2.06")]
din, dout = int(os.environ.get("DIN", 8192)), int(os.environ.get("DOUT", 28672))
m = P.DeviceModel.upload(random_packed(dout, din, fam, 64, 3))
for M in [int(v) for v in os.environ.get("MS", "5,6,7,8").split(",")]:
    x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
    y = P.matmul(m, x, kernel="gemv")
    torch.cuda.synchronize()
    ref = P.matmul(m, x, kernel="gemm")
    torch.cuda.synchronize()
    err = ((y - ref).norm() / ref.norm()).item()
    print(f"M={M} ok rel diff vs gemm {err:.2e}", flush=True)
