"""GPU quantizer (ccq_quantize_host) vs the reference quantize_tensor on all
host threads: a 1024 x 4096 slab per family, rounds = 2, sections compared."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2507_07145_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
w = (rng.standard_normal((1024, 4096)) * 0.02).astype(np.float32)
P.quantize(w[:8], 0)  # context
for name in ("2.75", "2.5", "2.06"):
    fam = P.FAMILIES[name]
    rows = 1024 if name != "2.06" else 256
    t0 = time.perf_counter()
    got = P.quantize(w[:rows], fam, 64, 2)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = O.RefModel.quantize(w[:rows], fam, 64, 2, threads=0).sections()
    tc = time.perf_counter() - t0
    same = np.array_equal(got.code_payload, want.code_payload) and np.array_equal(got.super_scales, want.super_scales)
    print(f"{name}: {rows}x4096 GPU {tg:7.3f} s ({rows * 4096 / tg / 1e6:8.2f} Mw/s) | reference {os.cpu_count()} threads "
          f"{tc:7.3f} s ({rows * 4096 / tc / 1e6:7.3f} Mw/s) | x{tc / tg:.1f} | sections equal: {same}")
