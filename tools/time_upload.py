"""Upload (load -> device layout) time for configs[4]'s 8192 -> 28672 layer, all families."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

if os.environ.get("CCQ_LIB"):  # experiment builds (tools only)
    P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ["CCQ_LIB"])
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

torch.cuda.init()
for name, fam in (("2.06", 2), ("2.75", 0), ("2.5", 1)):
    pm = random_packed(28672, 8192, fam, 64, 3)
    P.DeviceModel.upload(pm)  # warm (context, pools)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        d = P.DeviceModel.upload(pm)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del d
    mb = pm.payload_bytes / 1e6 if hasattr(pm, "payload_bytes") else 0
    print(f"{name}: upload {1e3 * min(ts):7.1f} ms  ({os.environ.get('CCQ_LIB', 'libccq_b200.so')})")
