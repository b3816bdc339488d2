"""Per-launch GEMV time: graph replay vs plain stream launches (is PDL overlap kept in graphs?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "2.06"]
ms = [P.DeviceModel.upload(random_packed(14336, 4096, fam, 64, 7 + c)) for c in range(20)]
x = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
ys = [torch.empty(1, 14336, device="cuda") for _ in ms]
s = torch.cuda.Stream()


def body():
    for m, y in zip(ms, ys):
        P.matmul(m, x, out=y, stream=s)


with torch.cuda.stream(s):
    body()
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(10):
        body()
    e1.record(s)
torch.cuda.synchronize()
print(f"stream launches: {e0.elapsed_time(e1) * 1e3 / (10 * len(ms)):.2f} us/launch")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    body()
g.replay()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
torch.cuda.synchronize()
print(f"graph replay:    {e0.elapsed_time(e1) * 1e3 / (10 * len(ms)):.2f} us/launch")
