import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_07145_b200 as P
from paper_2507_07145_b200.synthetic import random_packed
s = torch.cuda.Stream()
for fname in ("2.5", "2.75", "2.06"):
    ms = [P.DeviceModel.upload(random_packed(4096, 14336, P.FAMILIES[fname], 64, 3 + c)) for c in range(10)]
    for M in (2, 4, 8, 16):
        x = torch.randn(M, 14336, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, 4096, device="cuda")
        for kern in ("auto", "gemm"):
            def body():
                for m in ms:
                    P.matmul(m, x, out=y, stream=s, kernel=kern)
            with torch.cuda.stream(s):
                body()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(5):
                    body()
                e1.record(s)
            torch.cuda.synchronize()
            print(f"{fname} 14336x4096 M={M} {kern}: {e0.elapsed_time(e1) * 1e3 / 50:.1f} us")
