"""Host-side cost per matmul call (M=1, 4096 -> 14336): the Python wrapper vs
a bare ctypes call vs the C ABI alone (measured by issuing N calls and timing
the host before synchronising)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

m = P.DeviceModel.upload(random_packed(14336, 4096, 2, 64, 3))
x = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
y = torch.empty(1, 14336, device="cuda")
s = torch.cuda.Stream()
N = 2000
for _ in range(50):
    P.matmul(m, x, out=y, stream=s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    P.matmul(m, x, out=y, stream=s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"P.matmul: host {1e6 * (t1 - t0) / N:.2f} us/call, total {1e6 * (t2 - t0) / N:.2f} us/call")
fn = P.lib().ccq_cuda_matmul
args = (m.h, x.data_ptr(), 1, 1, y.data_ptr(), 0, C.c_void_p(s.cuda_stream))
t0 = time.perf_counter()
for _ in range(N):
    fn(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"bare ctypes: host {1e6 * (t1 - t0) / N:.2f} us/call, total {1e6 * (t2 - t0) / N:.2f} us/call")
