"""Launch one CCQ kernel a few times for ncu (not a benchmark).

  python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --M 1 --kernel gemv --reps 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="2.06")
ap.add_argument("--din", type=int, default=4096)
ap.add_argument("--dout", type=int, default=14336)
ap.add_argument("--M", type=int, default=1)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--copies", type=int, default=4)
ap.add_argument("--decode", action="store_true")
a = ap.parse_args()
fam = P.FAMILIES[a.family]
ms = [P.DeviceModel.upload(random_packed(a.dout, a.din, fam, 64, 3 + c)) for c in range(a.copies)]
x = torch.randn(a.M, a.din, device="cuda").to(torch.bfloat16)
y = torch.empty(a.M, a.dout, device="cuda")
if a.decode:
    w = torch.empty(a.dout, a.din, device="cuda")
    lv = torch.empty(a.dout, a.din, dtype=torch.int8, device="cuda")
for r in range(a.reps):
    for m in ms:
        if a.decode:
            P.decode(m, levels=lv, weights=w)
        else:
            P.matmul(m, x, out=y, kernel=a.kernel)
torch.cuda.synchronize()
print("done", P.launch_count())
