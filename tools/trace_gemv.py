"""Per-warp timeline of the streaming GEMV (debug build libccq_b200_trace.so)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_07145_b200 as P  # noqa: E402

P.LIB_PATH = os.path.join(os.path.dirname(P.__file__), "libccq_b200_trace.so")
import torch  # noqa: E402

from paper_2507_07145_b200.synthetic import random_packed  # noqa: E402

fam = P.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "2.06"]
din, dout = int(sys.argv[2]) if len(sys.argv) > 2 else 4096, int(sys.argv[3]) if len(sys.argv) > 3 else 14336
ms = [P.DeviceModel.upload(random_packed(dout, din, fam, 64, 3 + c)) for c in range(4)]
x = torch.randn(1, din, device="cuda").to(torch.bfloat16)
y = torch.empty(1, dout, device="cuda")
for r in range(3):
    for m in ms:
        P.matmul(m, x, out=y)
torch.cuda.synchronize()
buf = np.zeros(8192 * 16, np.uint64)
assert P.lib().ccq_trace_dump(C.c_void_p(buf.ctypes.data), buf.size) == 0
t = buf.reshape(8192, 16).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
base = t[:, 0].min()
cols = [0, 6, 7, 8, 9, 10, 11, 1, 2, 3, 4]
rel = (t[:, cols] - base) / 1000.0  # us
print("warps", used.sum())
names = ["start", "griddep ok", "x arrived", "tiles issued", "conv done", "conv sync", "Q done", "x ready", "first data", "loop end", "exit"]
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:10s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
print("tiles per warp: min", t[:, 5].min(), "max", t[:, 5].max(), "mean", t[:, 5].mean())
loop = rel[:, 9] - rel[:, 8]
print(f"loop time per warp: p50 {np.median(loop):.2f} max {loop.max():.2f} us; per tile p50 {np.median(loop / np.maximum(t[:, 5], 1)):.3f} us")

# per-CTA view: slowest warp loop end per CTA vs SM id (die locality / imbalance)
wpc = int(os.environ.get("WPC", "16"))
nct = t.shape[0] // wpc
cta_end = rel[: nct * wpc, 9].reshape(nct, wpc).max(1)
cta_first = rel[: nct * wpc, 8].reshape(nct, wpc).min(1)
smid = t[: nct * wpc, 12].reshape(nct, wpc)[:, 0]
order = np.argsort(smid)
print("CTA loop-end (max over warps) by SM id, us:")
print(" ".join(f"{int(smid[i])}:{cta_end[i]:.1f}" for i in order))
lo = smid < 74
print(f"SM<74 mean end {cta_end[lo].mean():.2f} max {cta_end[lo].max():.2f}; SM>=74 mean {cta_end[~lo].mean():.2f} max {cta_end[~lo].max():.2f}")
print(f"first data by SM half: {cta_first[lo].mean():.2f} / {cta_first[~lo].mean():.2f}")
# row-balance tail: CTAs whose slowest stream has one more tile (97- vs 96-row CTAs)
cta_tiles = t[: nct * wpc, 5].reshape(nct, wpc).max(1)
for k in np.unique(cta_tiles):
    sel = cta_tiles == k
    print(f"CTAs with max {int(k)} tiles/warp: {int(sel.sum())}, loop-end mean {cta_end[sel].mean():.2f} max {cta_end[sel].max():.2f}")
wt = t[:, 5]
for k in np.unique(wt):
    sel = wt == k
    print(f"warps with {int(k)} tiles: {int(sel.sum())}, loop end p50 {np.median(rel[sel, 9]):.2f}, loop time p50 {np.median(loop[sel]):.2f}")
# last / penultimate tile timing (slots 15 = penultimate tile data ready, 13 = last tile data ready, 14 = last tile done)
pen = (t[:, 15] - base) / 1000.0
lst = (t[:, 13] - base) / 1000.0
lend = (t[:, 14] - base) / 1000.0
for k in np.unique(wt):
    sel = wt == k
    print(f"{int(k)}-tile warps: penult start p50 {np.median(pen[sel]):.2f}, last start p50 {np.median(lst[sel]):.2f}, "
          f"last end p50 {np.median(lend[sel]):.2f}; last tile dur p50 {np.median(lend[sel] - lst[sel]):.3f}, "
          f"penult tile dur p50 {np.median(lst[sel] - pen[sel]):.3f}")
