"""Small end-to-end run of every kernel family for compute-sanitizer (tests/test_sanitizer.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2507_07145_b200 as P  # noqa: E402

for fam in (2, 0, 1):
    s = O.random_packed(160, 1024 + 64, fam, 64, seed=3 + fam)
    d = P.DeviceModel.upload(P.PackedModel.from_sections(s))
    lv = torch.empty(160, 1088, dtype=torch.int8, device="cuda")
    w = torch.empty(160, 1088, dtype=torch.float32, device="cuda")
    P.decode(d, levels=lv, weights=w)
    for M in (1, 3, 40):
        x = torch.from_numpy(O.random_matrix(M, 1088, "gaussian", M)).cuda().to(torch.bfloat16)
        P.matmul(d, x)
        P.matmul(d, x, kernel="gemm")
        P.matmul(d, x.float())
    secs = [O.random_packed(48, 1088, fam, 64, seed=e) for e in range(4)]
    ex = P.Experts.upload([P.PackedModel.from_sections(t) for t in secs])
    offs = np.array([0, 1, 1, 3, 4], np.int32)
    P.experts_matmul(ex, offs, torch.from_numpy(O.random_matrix(4, 1088, "gaussian", 9)).cuda().to(torch.bfloat16))
    offs1 = np.array([0, 1, 1, 2, 3], np.int32)  # one token per routed expert: grouped streaming GEMV
    P.experts_matmul(ex, offs1, torch.from_numpy(O.random_matrix(3, 1088, "gaussian", 10)).cuda().to(torch.bfloat16))
    # sync-free MoE forward (token-tile prefix + tile-list grouped GEMM + combine)
    ids = torch.tensor([[0, 2], [3, 1], [2, 0]], dtype=torch.int32, device="cuda")
    P.moe_forward(ex, ids, torch.rand(3, 2, device="cuda"),
                  torch.from_numpy(O.random_matrix(3, 1088, "gaussian", 11)).cuda().to(torch.bfloat16))
    # K-heavy layer (> 2 K chunks): direct activation loads in the M = 1 GEMV; M = 8 tensor-pipe GEMV
    sk = O.random_packed(64, 64 * 96, fam, 64, seed=21 + fam)
    dk = P.DeviceModel.upload(P.PackedModel.from_sections(sk))
    for M in (1, 8):
        P.matmul(dk, torch.from_numpy(O.random_matrix(M, 64 * 96, "gaussian", M)).cuda().to(torch.bfloat16))
    # quantizer kernels (csrc/quantize.cu)
    wq = (np.random.default_rng(fam).standard_normal((4, 128)) * 0.02).astype(np.float32)
    P.quantize(wq, fam, 64, 1)
cfg = P.ENCODINGS["2.06"]
P.search_codes(torch.randn(40, 4, device="cuda"), torch.rand(40, dtype=torch.float64, device="cuda"), cfg, valid=3)
torch.cuda.synchronize()
print("sanitize case ok")
