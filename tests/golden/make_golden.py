"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run here (needs oracle/_ref/libccq_ref.so, i.e. /root/reference present):

    python tests/golden/make_golden.py

Writes, per family:
  acc512_<fam>.ccq      the acceptance fixture of acceptance_main.cpp:94-112:
                        quantize_tensor(random_matrix(512, 512, Gaussian,
                        20260815)) written by ccq::write_container
  acc512_<fam>.npz      reference outputs on that model:
                        recon_sha  sha256 of ccq::reconstruct (quantizer side)
                        deq_sha    sha256 of ccq::dequantize
                        lv_sha     sha256 of centered levels (decode_group_states)
                        x, y       x = random_matrix(4, 512, Uniform, 516+m...) and
                                   y = ccq::gemv_batch(model, x)
  rand_<fam>_<shape>.npz  synthetic random_quantized models at
                        small sizes with their reference dequantize hash
and golden.json with the hashes (the tests read only the committed files).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

FAMS = {"2.75": 0, "2.5": 1, "2.06": 2}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    O.build(ref=True)
    out = {"acceptance": {}, "random": {}}
    w = O.ref_random_matrix(512, 512, "gaussian", 20260815)
    assert np.array_equal(w.view(np.uint32), O.random_matrix(512, 512, "gaussian",
                                                             20260815).view(np.uint32))
    for name, fam in FAMS.items():
        model, recon = O.RefModel.quantize(w, fam, 64, rounds=2, threads=0, want_recon=True)
        path = os.path.join(HERE, f"acc512_{name}.ccq")
        model.write(path)
        back = O.RefModel.load(path)
        deq = back.dequantize()
        assert np.array_equal(deq.view(np.uint32), recon.view(np.uint32)), "criterion 6"
        lv = back.levels()
        x = O.ref_random_matrix(4, 512, "uniform", 512 + 512 + 4)
        y = back.gemv_batch(x)
        np.savez_compressed(os.path.join(HERE, f"acc512_{name}.npz"), x=x, y=y)
        out["acceptance"][name] = {"recon_sha": sha(recon), "deq_sha": sha(deq),
                                   "lv_sha": sha(lv), "payload_bytes": back.payload_bytes()}
        print(name, "acceptance fixture", os.path.getsize(path), "bytes")
    for name, fam in FAMS.items():
        for (rows, cols, gs, seed) in [(96, 128, 64, 5), (33, 320, 64, 11), (8, 4096, 64, 7)]:
            m = O.RefModel.random(rows, cols, fam, gs, seed)
            deq = m.dequantize()
            lv = m.levels()
            key = f"{name}_{rows}x{cols}_g{gs}_s{seed}"
            x = O.ref_random_matrix(3, cols, "gaussian", seed + 1)
            y = m.gemv_batch(x)
            out["random"][key] = {"family": fam, "rows": rows, "cols": cols, "group_size": gs,
                                  "seed": seed, "deq_sha": sha(deq), "lv_sha": sha(lv),
                                  "y_sha": sha(y), "payload_bytes": m.payload_bytes()}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote golden.json")


if __name__ == "__main__":
    main()
