"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two libraries live here:

* ``_build/libccq_oracle.so`` — our plain-C restatement of the reference
  decode/GEMV path (``ccq_oracle.c``; every function cites the reference
  file:line it follows).  Always buildable (gcc), travels to the GPU box.
* ``_ref/libccq_ref.so`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/core/src`` plus ``ref_shim.cpp`` (built here only,
  git-ignored, but shipped to the GPU box with the snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
/ ``--impl reference`` legs may import this package, and only as the checker
or the timed reference; the product path never does.

Models are duck-typed: any object with ``rows, cols, family, group_size,
code_payload, scale_payload, super_scales, cluster_scales,
cluster_zero_points`` (numpy arrays for the sections) works.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libccq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libccq_ref.so")

FAMILIES = {"2.75": 0, "2.5": 1, "2.06": 2}
FAMILY_NAMES = {v: k for k, v in FAMILIES.items()}

STATUS = {0: None, 1: "ConfigError", 2: "DomainError", 3: "ShapeError",
          4: "EncodingError", 5: "FormatError", 9: "Error"}


class OracleError(Exception):
    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}" if msg else kind)
        self.kind = kind


def _check(st: int, msg: str = "") -> None:
    if st != 0:
        raise OracleError(STATUS.get(st, f"status {st}"), msg)


@dataclass
class Sections:
    """The five sections of ccq::PackedModel (container.hpp:37-52)."""
    rows: int
    cols: int
    family: int
    group_size: int
    code_payload: np.ndarray
    scale_payload: np.ndarray
    super_scales: np.ndarray
    cluster_scales: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    cluster_zero_points: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    rounds: int = 0


class _ModelView(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("family", C.c_int),
                ("group_size", C.c_int),
                ("code_payload", C.c_void_p), ("code_bytes", C.c_size_t),
                ("scale_payload", C.c_void_p), ("scale_bytes", C.c_size_t),
                ("super_scales", C.c_void_p), ("cluster_scales", C.c_void_p),
                ("cluster_zero_points", C.c_void_p)]


def _ptr(a: np.ndarray | None):
    if a is None or a.size == 0:
        return None
    return a.ctypes.data


def build(ref: bool = False) -> None:
    """Compile the C oracle (and, when /root/reference exists, the reference)."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        vp, i64, sz = C.c_void_p, C.c_int64, C.c_size_t
        L.ccqo_dequantize.argtypes = [C.POINTER(_ModelView), vp]
        L.ccqo_levels.argtypes = [C.POINTER(_ModelView), vp]
        L.ccqo_group_scales.argtypes = [C.POINTER(_ModelView), vp]
        L.ccqo_gemv_batch.argtypes = [C.POINTER(_ModelView), vp, i64, vp]
        L.ccqo_gemv_batch_mt.argtypes = [C.POINTER(_ModelView), vp, i64, vp, C.c_int]
        L.ccqo_payload_bytes.argtypes = [C.POINTER(_ModelView)]
        L.ccqo_payload_bytes.restype = C.c_uint64
        L.ccqo_validate.argtypes = [C.POINTER(_ModelView)]
        L.ccqo_random_matrix.argtypes = [i64, i64, C.c_int, C.c_uint64, vp]
        L.ccqo_random_matrix.restype = None
        L.ccqo_section_sizes.argtypes = [i64, i64, C.c_int, C.c_int, C.POINTER(sz),
                                         C.POINTER(sz), C.POINTER(sz)]
        L.ccqo_random_packed.argtypes = [i64, i64, C.c_int, C.c_int, C.c_uint64,
                                         vp, vp, vp, vp, vp]
        L.ccqo_clustered_code_value.argtypes = [C.c_uint8, C.c_float, C.c_float, C.c_int,
                                                C.POINTER(C.c_uint16)]
        L.ccqo_group_geometry.argtypes = [C.c_int, C.c_int, vp]
        L.ccqo_pack_cluster_scales.argtypes = [vp, sz, vp]
        L.ccqo_unpack_cluster_scales.argtypes = [vp, sz, sz, vp]
        L.ccqo_pack_group.argtypes = [vp, sz, C.c_uint16, C.c_int, C.c_int, vp,
                                      C.POINTER(C.c_uint16)]
        _lib = L
    return _lib


def _view(m) -> _ModelView:
    arrs = [np.ascontiguousarray(m.code_payload, np.uint8),
            np.ascontiguousarray(m.scale_payload, np.uint8),
            np.ascontiguousarray(m.super_scales, np.float32),
            np.ascontiguousarray(m.cluster_scales, np.float32),
            np.ascontiguousarray(m.cluster_zero_points, np.float32)]
    v = _ModelView(int(m.rows), int(m.cols), int(m.family), int(m.group_size),
                   _ptr(arrs[0]), arrs[0].size, _ptr(arrs[1]), arrs[1].size,
                   _ptr(arrs[2]), _ptr(arrs[3]), _ptr(arrs[4]))
    v._keep = arrs  # keep buffers alive with the view
    return v


# ---------------------------------------------------------------- oracle --

def section_sizes(rows, cols, family, group_size):
    a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
    _check(lib().ccqo_section_sizes(rows, cols, family, group_size, a, b, c))
    return a.value, b.value, c.value


def random_packed(rows, cols, family, group_size=64, seed=1) -> Sections:
    """pack_model(random_quantized(...)) restated (synthetic.cpp:25-103)."""
    cb, sb, cr = section_sizes(rows, cols, family, group_size)
    code = np.zeros(cb, np.uint8)
    scale = np.zeros(sb, np.uint8)
    sup = np.zeros(rows, np.float32)
    cs = np.zeros(cr, np.float32)
    czp = np.zeros(cr, np.float32)
    _check(lib().ccqo_random_packed(rows, cols, family, group_size, seed, _ptr(code),
                                    _ptr(scale), _ptr(sup), _ptr(cs), _ptr(czp)))
    return Sections(rows, cols, family, group_size, code, scale, sup, cs, czp)


def random_matrix(rows, cols, dist="gaussian", seed=1) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    lib().ccqo_random_matrix(rows, cols, 0 if dist == "gaussian" else 1, seed, _ptr(out))
    return out


def dequantize(m) -> np.ndarray:
    out = np.empty((m.rows, m.cols), np.float32)
    _check(lib().ccqo_dequantize(C.byref(_view(m)), _ptr(out)))
    return out


def levels(m) -> np.ndarray:
    out = np.empty((m.rows, m.cols), np.int8)
    _check(lib().ccqo_levels(C.byref(_view(m)), _ptr(out)))
    return out


def group_scales(m) -> np.ndarray:
    out = np.empty((m.rows, m.cols // m.group_size), np.float32)
    _check(lib().ccqo_group_scales(C.byref(_view(m)), _ptr(out)))
    return out


def gemv_batch(m, x: np.ndarray, threads: int = 1) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    x = x.reshape(1, -1) if x.ndim == 1 else x
    y = np.empty((x.shape[0], m.rows), np.float32)
    if threads > 1:
        _check(lib().ccqo_gemv_batch_mt(C.byref(_view(m)), _ptr(x), x.shape[0], _ptr(y),
                                        threads))
    else:
        _check(lib().ccqo_gemv_batch(C.byref(_view(m)), _ptr(x), x.shape[0], _ptr(y)))
    return y


def payload_bytes(m) -> int:
    return int(lib().ccqo_payload_bytes(C.byref(_view(m))))


def validate(m) -> None:
    _check(lib().ccqo_validate(C.byref(_view(m))))


def clustered_code_value(q, alpha, beta, code_bits=15) -> int:
    out = C.c_uint16()
    _check(lib().ccqo_clustered_code_value(q, alpha, beta, code_bits, C.byref(out)))
    return out.value


def group_geometry(family, group_size) -> dict:
    g = (C.c_int * 6)()
    _check(lib().ccqo_group_geometry(family, group_size, g))
    keys = ("group_size", "full_words", "has_tail", "words_per_group", "embedded_scale",
            "payload_bytes")
    return dict(zip(keys, list(g)))


def pack_cluster_scales(codes) -> bytes:
    c = np.ascontiguousarray(codes, np.uint16)
    out = np.zeros((c.size + 1) // 2, np.uint8)
    _check(lib().ccqo_pack_cluster_scales(_ptr(c), c.size, _ptr(out)))
    return out.tobytes()


def unpack_cluster_scales(data: bytes, count: int) -> list:
    b = np.frombuffer(bytes(data), np.uint8).copy()
    out = np.zeros(count, np.uint16)
    _check(lib().ccqo_unpack_cluster_scales(_ptr(b), b.size, count, _ptr(out)))
    return out.tolist()


def pack_group(codes, scale_code, family, group_size=64):
    c = np.ascontiguousarray(codes, np.uint16)
    g = group_geometry(family, group_size)
    out = np.zeros(g["payload_bytes"], np.uint8)
    side = C.c_uint16()
    _check(lib().ccqo_pack_group(_ptr(c), c.size, scale_code, family, group_size, _ptr(out),
                                 C.byref(side)))
    return out.tobytes(), side.value


# ------------------------------------------------------------- reference --

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The unmodified reference library (oracle/_ref/libccq_ref.so)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        vp, i64, u64 = C.c_void_p, C.c_int64, C.c_uint64
        L.ccqref_last_error.restype = C.c_char_p
        L.ccqref_free.argtypes = [vp]
        L.ccqref_free.restype = None
        L.ccqref_model_random.argtypes = [i64, i64, C.c_int, C.c_int, u64, C.POINTER(vp)]
        L.ccqref_model_quantize.argtypes = [vp, i64, i64, C.c_int, C.c_int, C.c_int, C.c_int,
                                            vp, C.POINTER(vp)]
        L.ccqref_model_from_sections.argtypes = [i64, i64, C.c_int, C.c_int, C.c_int, vp,
                                                 C.c_size_t, vp, C.c_size_t, vp, vp, vp,
                                                 C.POINTER(vp)]
        L.ccqref_load_model.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ccqref_search_codes.argtypes = [vp, i64, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.ccqref_write_container.argtypes = [vp, C.c_char_p]
        L.ccqref_model_shape.argtypes = [vp] + [C.POINTER(i64)] * 2 + [C.POINTER(C.c_int)] * 3 \
            + [C.POINTER(u64)] * 3
        L.ccqref_model_shape.restype = None
        L.ccqref_model_sections.argtypes = [vp] * 6
        L.ccqref_model_sections.restype = None
        L.ccqref_payload_bytes.argtypes = [vp]
        L.ccqref_payload_bytes.restype = u64
        L.ccqref_dequantize.argtypes = [vp, vp]
        L.ccqref_levels.argtypes = [vp, vp]
        L.ccqref_gemv.argtypes = [vp, vp, vp]
        L.ccqref_gemv_batch.argtypes = [vp, vp, i64, vp]
        L.ccqref_sliced_new.argtypes = [vp, C.c_int, vp]
        L.ccqref_gemv_batch_parts.argtypes = [vp, C.c_int, vp, i64, vp, i64]
        L.ccqref_random_matrix.argtypes = [i64, i64, C.c_int, u64, vp]
        L.ccqref_random_matrix.restype = None
        L.ccqref_clustered_code_value.argtypes = [C.c_uint8, C.c_float, C.c_float, C.c_int,
                                                  C.POINTER(C.c_uint16)]
        L.ccqref_group_geometry.argtypes = [C.c_int, C.c_int, vp]
        _ref = L
    return _ref


def _rcheck(st):
    if st != 0:
        raise OracleError(STATUS.get(st, f"status {st}"), ref().ccqref_last_error().decode())


class RefModel:
    """Owning handle to a reference ccq::PackedModel."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ccqref_free(self.h)
            self.h = None

    @staticmethod
    def random(rows, cols, family, group_size=64, seed=1) -> "RefModel":
        h = C.c_void_p()
        _rcheck(ref().ccqref_model_random(rows, cols, family, group_size, seed, C.byref(h)))
        return RefModel(h)

    @staticmethod
    def quantize(w: np.ndarray, family, group_size=64, rounds=2, threads=0,
                 want_recon=False):
        w = np.ascontiguousarray(w, np.float32)
        recon = np.empty_like(w) if want_recon else None
        h = C.c_void_p()
        _rcheck(ref().ccqref_model_quantize(_ptr(w), w.shape[0], w.shape[1], family,
                                            group_size, rounds, threads, _ptr(recon),
                                            C.byref(h)))
        return (RefModel(h), recon) if want_recon else RefModel(h)

    @staticmethod
    def from_sections(m) -> "RefModel":
        v = _view(m)
        h = C.c_void_p()
        _rcheck(ref().ccqref_model_from_sections(
            int(m.rows), int(m.cols), int(m.family), int(m.group_size),
            int(getattr(m, "rounds", 0)), v.code_payload, v.code_bytes, v.scale_payload,
            v.scale_bytes, v.super_scales, v.cluster_scales, v.cluster_zero_points,
            C.byref(h)))
        return RefModel(h)

    @staticmethod
    def load(path: str) -> "RefModel":
        h = C.c_void_p()
        _rcheck(ref().ccqref_load_model(path.encode(), C.byref(h)))
        return RefModel(h)

    def write(self, path: str) -> None:
        _rcheck(ref().ccqref_write_container(self.h, path.encode()))

    def sections(self) -> Sections:
        r, c = C.c_int64(), C.c_int64()
        f, g, rd = C.c_int(), C.c_int(), C.c_int()
        cl, sl, kl = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ref().ccqref_model_shape(self.h, r, c, f, g, rd, cl, sl, kl)
        code = np.zeros(cl.value, np.uint8)
        scale = np.zeros(sl.value, np.uint8)
        sup = np.zeros(r.value, np.float32)
        cs = np.zeros(kl.value, np.float32)
        czp = np.zeros(kl.value, np.float32)
        ref().ccqref_model_sections(self.h, _ptr(code), _ptr(scale), _ptr(sup), _ptr(cs),
                                    _ptr(czp))
        return Sections(r.value, c.value, f.value, g.value, code, scale, sup, cs, czp,
                        rounds=rd.value)

    def payload_bytes(self) -> int:
        return int(ref().ccqref_payload_bytes(self.h))

    def dequantize(self) -> np.ndarray:
        s = self.sections()
        out = np.empty((s.rows, s.cols), np.float32)
        _rcheck(ref().ccqref_dequantize(self.h, _ptr(out)))
        return out

    def levels(self) -> np.ndarray:
        s = self.sections()
        out = np.empty((s.rows, s.cols), np.int8)
        _rcheck(ref().ccqref_levels(self.h, _ptr(out)))
        return out

    def gemv_batch(self, x: np.ndarray) -> np.ndarray:
        s = self.sections()
        x = np.ascontiguousarray(x, np.float32)
        x = x.reshape(1, -1) if x.ndim == 1 else x
        y = np.empty((x.shape[0], s.rows), np.float32)
        _rcheck(ref().ccqref_gemv_batch(self.h, _ptr(x), x.shape[0], _ptr(y)))
        return y

    def gemv(self, x: np.ndarray) -> np.ndarray:
        s = self.sections()
        x = np.ascontiguousarray(x, np.float32).reshape(s.cols)
        y = np.empty(s.rows, np.float32)
        _rcheck(ref().ccqref_gemv(self.h, _ptr(x), _ptr(y)))
        return y


class RefSharded:
    """The reference gemv_batch over contiguous row blocks, one std::thread
    each (the all-cores CPU baseline of SURVEY §8d)."""

    def __init__(self, model: RefModel, parts: int):
        s = model.sections()
        self.rows, self.cols = s.rows, s.cols
        parts = max(1, min(parts, s.rows))
        self.handles = (C.c_void_p * parts)()
        _rcheck(ref().ccqref_sliced_new(model.h, parts, self.handles))
        self.parts = parts

    def __del__(self):
        if _ref is not None:
            for h in self.handles:
                if h:
                    _ref.ccqref_free(h)

    def gemv_batch(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        x = x.reshape(1, -1) if x.ndim == 1 else x
        y = np.empty((x.shape[0], self.rows), np.float32)
        _rcheck(ref().ccqref_gemv_batch_parts(self.handles, self.parts, _ptr(x), x.shape[0],
                                              _ptr(y), self.rows))
        return y


def ref_random_matrix(rows, cols, dist="gaussian", seed=1) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    ref().ccqref_random_matrix(rows, cols, 0 if dist == "gaussian" else 1, seed, _ptr(out))
    return out


def ref_clustered_code_value(q, alpha, beta, code_bits=15) -> int:
    out = C.c_uint16()
    _rcheck(ref().ccqref_clustered_code_value(q, alpha, beta, code_bits, C.byref(out)))
    return out.value
