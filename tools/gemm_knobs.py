"""One GEMM timing for tuning experiments (env knobs CCQ_GEMM_BN,
CCQ_GEMM_SPLITS, CCQ_GROUPED_BN are read once per process):

  python tools/gemm_knobs.py dense FAMILY D_IN D_OUT M
  python tools/gemm_knobs.py moe ernie|deepseek [T]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

peak = float(bench.load_peaks().get("bf16_tflops", 1679.5))
s = torch.cuda.Stream()
knobs = {k: os.environ[k] for k in ("CCQ_GEMM_BN", "CCQ_GEMM_SPLITS", "CCQ_GROUPED_BN", "CCQ_GEMM_SK", "CCQ_GEMM_PAR", "CCQ_GEMM_RT") if k in os.environ}
if sys.argv[1] == "dense":
    fam, din, dout, M = P.FAMILIES[sys.argv[2]], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    copies = max(2, int(160e6 // (din * dout * 0.3)) + 1)
    ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 40 + c)) for c in range(copies)]
    x = torch.randn(M, din, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, dout, device="cuda")
    kern = os.environ.get("KNOB_KERNEL")  # force a path ("gemm", ...) instead of the dispatch
    if kern:
        knobs["KNOB_KERNEL"] = kern
        us = bench._graph_time_us(torch, s, lambda: [P.matmul(mm, x, out=y, stream=s, kernel=kern) for mm in ms],
                                  reps=10) / len(ms)
    else:
        us = bench._l2_cold_us(P, torch, None, s, ms, x, y)
    tf = 2 * M * din * dout / us / 1e6
    print(json.dumps({"case": "dense", "family": sys.argv[2], "d_in": din, "d_out": dout, "M": M, "knobs": knobs,
                      "us": round(us, 2), "TFLOPs": round(tf, 1), "tensor_frac": round(tf / peak, 4)}))
else:
    name = sys.argv[2]
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
    E, din, dout = (64, 8192, 3584) if name == "ernie" else (256, 7168, 2048)
    ex = P.Experts.upload([random_packed(dout, din, 2, 64, 1000 + e) for e in range(E)])
    rng = np.random.default_rng(7)
    counts = np.zeros(E, np.int64)
    for _ in range(T):
        counts[rng.choice(E, 8, replace=False)] += 1
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    pairs = int(offs[-1])
    offs_dev = torch.from_numpy(offs).cuda()
    x = torch.randn(pairs, din, device="cuda").to(torch.bfloat16)
    y = torch.empty(pairs, dout, device="cuda", dtype=torch.bfloat16)
    us = bench._graph_time_us(torch, s, lambda: P.experts_matmul(ex, offs, x, out=y, stream=s, offsets_dev=offs_dev),
                              reps=5)
    tf = 2 * pairs * din * dout / us / 1e6
    print(json.dumps({"case": "moe", "model": name, "T": T, "max_tokens": int(counts.max()),
                      "mean_tokens": float(counts.mean()), "knobs": knobs, "us": round(us, 1), "TFLOPs": round(tf, 1),
                      "tensor_frac": round(tf / peak, 4)}))
