"""Synthetic packed models for benchmarks.

`reference_packed` is the reference bench generator itself
(pack_model(random_quantized(...)), synthetic.cpp:25-103, the same
std::mt19937_64 stream; C++ in libccq_b200.so, ccq_synthetic_packed): a seed
gives the reference's exact bytes, so the GPU arm and the reference CPU arm
of bench.py time identical weights.

`random_packed` (numpy, vectorised, faster for big sweeps) draws the same
distribution - uniform stored code words, uniform scale codes in
[0, 2^scale_bits), super scales ~ U[0.001, 0.051), and for the clustered
family alpha ~ U[1, 1+32767/512), beta ~ U[0, 32767 - 255 alpha) - from
numpy's stream, so its bytes differ from the reference's for a seed.
"""
from __future__ import annotations

import numpy as np

from . import PackedModel, group_geometry

_WPW = {0: 3, 1: 7, 2: 4}
_STATE_BITS = {0: 4, 1: 3, 2: 6}
_SCALE_BITS = {0: 4, 1: 13, 2: 4}
_WORD_BITS = {0: 8, 1: 16, 2: 16}


def random_packed(rows: int, cols: int, family: int, group_size: int = 64,
                  seed: int = 0) -> PackedModel:
    rng = np.random.default_rng(seed)
    g = group_geometry(family, group_size)
    if cols % group_size:
        raise ValueError("cols must be a whole number of groups")
    groups = rows * (cols // group_size)
    wpg, full, pb = g["words_per_group"], g["full_words"], g["payload_bytes"]
    sup = (0.001 + 0.05 * rng.random(rows)).astype(np.float32)
    scale_codes = rng.integers(0, 1 << _SCALE_BITS[family], groups, dtype=np.uint32)
    cs = czp = np.zeros(0, np.float32)
    if family == 2:
        limit = 32767.0
        alpha = 1.0 + rng.random(rows) * (limit / 512.0)
        beta = rng.random(rows) * (limit - 255.0 * alpha)
        cs, czp = alpha.astype(np.float32), beta.astype(np.float32)
        codes = rng.integers(0, 256, (groups, pb), dtype=np.uint8)
        nib = np.zeros((groups + 1) // 2, np.uint8)
        sc = scale_codes.astype(np.uint8)
        nib[: groups // 2] = sc[0: 2 * (groups // 2): 2] | (sc[1: 2 * (groups // 2): 2] << 4)
        if groups % 2:
            nib[-1] = sc[-1]
        scale = nib
    elif family == 0:
        codes = rng.integers(0, 256, (groups, pb), dtype=np.uint8)
        if g["has_tail"]:
            st = rng.integers(0, 16, groups, dtype=np.uint8)
            codes[:, full] = (st << 4) | scale_codes.astype(np.uint8)
            scale = np.zeros(0, np.uint8)
        else:
            scale = _nibbles(scale_codes)
    else:
        words = rng.integers(0, 1 << 16, (groups, wpg), dtype=np.uint32)
        st = rng.integers(0, 8, groups, dtype=np.uint32)
        words[:, full] = (st << 13) | scale_codes
        codes = np.empty((groups, pb), np.uint8)
        codes[:, 0::2] = (words & 0xFF).astype(np.uint8)
        codes[:, 1::2] = (words >> 8).astype(np.uint8)
        scale = np.zeros(0, np.uint8)
    return PackedModel(rows, cols, family, group_size, codes.reshape(-1), scale, sup, cs, czp)


def reference_packed(rows: int, cols: int, family: int, group_size: int = 64, seed: int = 0) -> PackedModel:
    """The reference's random_quantized + pack_model bytes for `seed`."""
    from . import _check, _np_ptr, lib
    g = group_geometry(family, group_size)
    if cols % group_size:
        raise ValueError("cols must be a whole number of groups")
    groups = rows * (cols // group_size)
    code = np.empty(groups * g["payload_bytes"], np.uint8)
    scale = np.zeros(0 if g["embedded_scale"] else (groups + 1) // 2, np.uint8)
    sup = np.empty(rows, np.float32)
    cs = np.empty(rows if family == 2 else 0, np.float32)
    czp = np.empty(rows if family == 2 else 0, np.float32)
    _check(lib().ccq_synthetic_packed(rows, cols, family, group_size, seed, _np_ptr(code),
                                      _np_ptr(scale) if scale.size else None, _np_ptr(sup),
                                      _np_ptr(cs) if cs.size else None, _np_ptr(czp) if czp.size else None))
    return PackedModel(rows, cols, family, group_size, code, scale, sup, cs, czp)


def reference_matrix(rows: int, cols: int, dist: str = "gaussian", seed: int = 0) -> np.ndarray:
    """The reference's random_matrix (tensor.cpp:37-69) for `seed`, f32."""
    from . import _check, _np_ptr, lib
    out = np.empty((rows, cols), np.float32)
    _check(lib().ccq_synthetic_matrix(rows, cols, 0 if dist == "gaussian" else 1, seed,
                                      _np_ptr(out) if out.size else None))
    return out


def _nibbles(codes: np.ndarray) -> np.ndarray:
    n = codes.size
    c = codes.astype(np.uint8)
    out = np.zeros((n + 1) // 2, np.uint8)
    out[: n // 2] = c[0: 2 * (n // 2): 2] | (c[1: 2 * (n // 2): 2] << 4)
    if n % 2:
        out[-1] = c[-1]
    return out
