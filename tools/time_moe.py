"""Run bench.py's MoE section alone (configs[2]/[3] decode batches)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_07145_b200 as P  # noqa: E402

if os.environ.get("CCQ_LIB"):  # experiment builds (tools only)
    P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), os.environ["CCQ_LIB"])

peaks = bench.load_peaks()
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
for r in bench.run_moe(P, torch, dev, s, float(peaks.get("hbm_gbs", 6650)), float(peaks.get("bf16_tflops", 1590))):
    print(json.dumps(r))
