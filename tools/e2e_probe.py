"""Where does the e2e step time go?  12 rotating 4096 -> 14336 layers, M=1:
graph replay vs eager P.matmul (no copies) vs eager with H2D/D2H."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

L = 12
layers = [P.DeviceModel.upload(random_packed(14336, 4096, 2, 64, 3 + i)) for i in range(L)]
xh = torch.randn(L, 1, 4096).to(torch.bfloat16).pin_memory()
xd = xh.cuda()
yd = torch.empty(L, 1, 14336, device="cuda")
yh = torch.empty(L, 1, 14336).pin_memory()
s = torch.cuda.Stream()


def timeit(fn, steps=50):
    with torch.cuda.stream(s):
        for _ in range(5):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(steps):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


def compute():
    for l in range(L):
        P.matmul(layers[l], xd[l], out=yd[l], stream=s)


def with_copies():
    xd.copy_(xh, non_blocking=True)
    compute()
    yh.copy_(yd, non_blocking=True)


g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    compute()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    compute()
print(f"graph replay      : {timeit(g.replay):7.1f} us/step")
print(f"eager, no copies  : {timeit(compute):7.1f} us/step")
print(f"eager + H2D + D2H : {timeit(with_copies):7.1f} us/step")
print("(bench.py overlaps the copies on two copy streams, double-buffered)")
