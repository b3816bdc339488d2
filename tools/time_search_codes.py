"""GPU exhaustive code search vs the reference's search_codes on the host
(one thread; the reference parallelises quantize_tensor over rows): weights
per second for each family's encoding (subvector = states_per_code weights)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2507_07145_b200 as P  # noqa: E402

L = O.ref()
for name, cfg in P.ENCODINGS.items():
    Lb, N, S = cfg
    zp = 1 << (Lb - 1)
    n_gpu = 1 << 20 if name != "2.06" else 1 << 17
    rng = np.random.default_rng(1)
    t = (rng.standard_normal((n_gpu, N)) * 0.02).astype(np.float32)
    sc = np.abs(t).max(axis=1).astype(np.float64) / (zp - 1)
    tg, sg = torch.from_numpy(t).cuda(), torch.from_numpy(sc).cuda()
    P.search_codes(tg[:1024], sg[:1024], cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    codes = P.search_codes(tg, sg, cfg)
    e1.record()
    torch.cuda.synchronize()
    g_s = e0.elapsed_time(e1) * 1e-3
    n_cpu = 2000 if name == "2.06" else 200000
    out = np.zeros(n_cpu, np.uint32)
    t0 = time.perf_counter()
    L.ccqref_search_codes(t.ctypes.data, n_cpu, N, N, sc.ctypes.data, zp, Lb, N, S, out.ctypes.data)
    c_s = time.perf_counter() - t0
    same = np.array_equal(codes[:n_cpu].cpu().numpy().astype(np.uint32), out)
    gw, cw = n_gpu * N / g_s / 1e6, n_cpu * N / c_s / 1e6
    print(f"{name:9s} (L,N,S)={cfg}: GPU {gw:10.1f} Mw/s ({n_gpu} subvectors, {1e3 * g_s:.2f} ms) | "
          f"reference 1 thread {cw:8.3f} Mw/s ({n_cpu} subvectors) | x{gw / cw:,.0f} | codes equal: {same}")
