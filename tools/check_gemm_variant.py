"""Consistency check for experiment builds: tcgen05 GEMM vs the GEMV paths
(all families, M = 16 / 64 / 300, 4096 -> 14336)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

if os.environ.get("CCQ_LIB"):
    P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ["CCQ_LIB"])
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

worst = 0.0
for name, fam in (("2.06", 2), ("2.75", 0), ("2.5", 1)):
    m = P.DeviceModel.upload(random_packed(14336, 4096, fam, 64, 9))
    for M in (16, 64, 300):
        x = torch.randn(M, 4096, device="cuda").to(torch.bfloat16)
        a = P.matmul(m, x, kernel="gemm")
        b = P.matmul(m, x, kernel="gemv")
        torch.cuda.synchronize()
        err = ((a - b).norm() / b.norm()).item()
        worst = max(worst, err)
        print(f"{name} M={M}: rel diff {err:.2e}")
print("OK" if worst < 1e-4 else "MISMATCH", worst)
