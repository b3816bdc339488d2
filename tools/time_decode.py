"""Standalone decode (kernel a) throughput: read-GB/s (packed payload) and
total-GB/s (payload + outputs written) per family at configs[1]
(4096 -> 14336), for f32 weights, int8 levels and both.  CUDA events over
graph-replayed launches rotating across model copies (L2-cold)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_07145_b200 as P  # noqa: E402
from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

din, dout = 4096, 14336
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6549.1)
s = torch.cuda.Stream()
for fname in ("2.06", "2.75", "2.5"):
    fam = P.FAMILIES[fname]
    ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 21 + c)) for c in range(4)]
    pb = ms[0].payload_bytes
    w = torch.empty(dout, din, device="cuda")
    lv = torch.empty(dout, din, dtype=torch.int8, device="cuda")
    for mode in ("weights", "levels", "both"):
        def body():
            for m in ms:
                P.decode(m, levels=lv if mode != "weights" else None, weights=w if mode != "levels" else None,
                         stream=s)
        with torch.cuda.stream(s):
            body()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * len(ms))
        wrote = dout * din * ({"weights": 4, "levels": 1, "both": 5}[mode])
        print(json.dumps({"family": fname, "d_in": din, "d_out": dout, "outputs": mode, "us": round(us, 2),
                          "read_GBps": round(pb / us / 1e3, 1),
                          "total_GBps": round((pb + wrote) / us / 1e3, 1),
                          "total_frac_hbm": round((pb + wrote) / us / 1e3 / peak, 3)}))
