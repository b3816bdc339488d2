"""B200-native CCQ hot path: Python mirror of the reference C++ API.

The product is ``libccq_b200.so`` (hand-written sm_100a CUDA + C++ host code
behind the C ABI in ``include/ccq_cuda.h``).  This module binds that ABI with
ctypes and mirrors the reference operator surface so tests read like the
reference's own (``/root/reference/proj/core/include/ccq/kernels.hpp:36-76``,
``container.hpp:37-99``):

* ``PackedModel``            - ccq::PackedModel (container.hpp:37-52), host sections
* ``load_model(path)``       - ccq::load_model (container.hpp:83)
* ``dequantize(model)``      - ccq::dequantize (kernels.hpp:36)
* ``gemv(model, x)``         - ccq::gemv (kernels.hpp:39)
* ``gemv_batch(model, X)``   - ccq::gemv_batch (kernels.hpp:43)
* ``model_payload_bytes``    - ccq::model_payload_bytes (kernels.hpp:51)
* ``group_geometry``, ``clustered_code_value`` (packing.hpp:49, coding.hpp:142)

plus the device-resident layer (``DeviceModel``, ``decode``, ``matmul``,
``grouped``) that works on torch CUDA tensors without host copies.

Errors are raised as the reference exception types (error.hpp:25-68).  There
is no CPU fallback: if the library or a GPU is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CcqError", "ConfigError", "DomainError", "ShapeError", "EncodingError", "FormatError",
    "CudaError", "FAMILIES", "PackedModel", "DeviceModel", "load_model", "dequantize", "gemv",
    "gemv_batch", "model_payload_bytes", "group_geometry", "clustered_code_value", "decode",
    "matmul", "grouped", "search_codes", "quantize", "quantize_to_device", "ENCODINGS", "lib", "LIB_PATH", "launch_count", "Experts", "experts_matmul",
    "moe_forward",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libccq_b200.so")

FAMILIES = {"2.75": 0, "2.5": 1, "2.06": 2}
DTYPES = {"f32": 0, "bf16": 1, "f16": 2}


class CcqError(RuntimeError):
    """ccq::Error (error.hpp:25)."""


class ConfigError(CcqError):
    pass


class DomainError(CcqError):
    pass


class ShapeError(CcqError):
    pass


class EncodingError(CcqError):
    pass


class FormatError(CcqError):
    pass


class CudaError(CcqError):
    pass


_STATUS = {1: ConfigError, 2: DomainError, 3: ShapeError, 4: EncodingError, 5: FormatError,
           6: CudaError, 7: CcqError}


class _View(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("family", C.c_int32),
                ("group_size", C.c_int32), ("rounds", C.c_int32), ("reserved", C.c_int32),
                ("code_payload", C.c_void_p), ("code_bytes", C.c_uint64),
                ("scale_payload", C.c_void_p), ("scale_bytes", C.c_uint64),
                ("super_scales", C.c_void_p), ("n_super_scales", C.c_uint64),
                ("cluster_scales", C.c_void_p), ("n_cluster_scales", C.c_uint64),
                ("cluster_zero_points", C.c_void_p), ("n_cluster_zero_points", C.c_uint64)]


class ModelInfo(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("family", C.c_int32),
                ("group_size", C.c_int32), ("rounds", C.c_int32), ("device", C.c_int32),
                ("payload_bytes_per_group", C.c_int32), ("embedded_scale", C.c_int32),
                ("payload_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
                ("code_row_stride", C.c_uint64), ("fast_path", C.c_int32),
                ("reserved", C.c_int32)]


# Every symbol include/ccq_cuda.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = [
    "ccq_cuda_last_error", "ccq_cuda_version", "ccq_cuda_model_upload", "ccq_cuda_model_load",
    "ccq_container_open", "ccq_container_close", "ccq_cuda_model_upload_rows",
    "ccq_cuda_model_free", "ccq_cuda_model_info", "ccq_cuda_decode", "ccq_cuda_matmul",
    "ccq_cuda_gemv", "ccq_cuda_gemm", "ccq_cuda_grouped", "ccq_dequantize_host",
    "ccq_gemv_host", "ccq_gemv_batch_host", "ccq_model_payload_bytes", "ccq_group_geometry",
    "ccq_clustered_code_value", "ccq_cuda_launch_count", "ccq_cuda_experts_upload",
    "ccq_cuda_experts_matmul", "ccq_cuda_moe_forward", "ccq_cuda_search_codes",
    "ccq_quantize_host", "ccq_cuda_quantize_model", "ccq_nccl_unique_id", "ccq_nccl_comm_init",
    "ccq_nccl_comm_destroy", "ccq_cuda_shard_allgather", "ccq_synthetic_packed", "ccq_synthetic_matrix",
]

_lib = None


def lib():
    """Load libccq_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() (no CPU "
                              "fallback exists for the CCQ hot path)")
        L = C.CDLL(LIB_PATH)
        vp, i64, u64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32
        L.ccq_cuda_last_error.restype = C.c_char_p
        L.ccq_cuda_version.restype = C.c_char_p
        L.ccq_cuda_launch_count.restype = u64
        L.ccq_cuda_model_upload.argtypes = [C.POINTER(_View), C.c_int, C.POINTER(vp)]
        L.ccq_cuda_model_upload_rows.argtypes = [C.POINTER(_View), i64, i64, C.c_int,
                                                 C.POINTER(vp)]
        L.ccq_cuda_model_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.ccq_container_open.argtypes = [C.c_char_p, C.POINTER(_View), C.POINTER(vp)]
        L.ccq_container_close.argtypes = [vp]
        L.ccq_container_close.restype = None
        L.ccq_cuda_model_free.argtypes = [vp]
        L.ccq_cuda_model_info.argtypes = [vp, C.POINTER(ModelInfo)]
        L.ccq_cuda_decode.argtypes = [vp, vp, vp, vp]
        for fn in (L.ccq_cuda_matmul, L.ccq_cuda_gemv, L.ccq_cuda_gemm):
            fn.argtypes = [vp, vp, C.c_int, i64, vp, C.c_int, vp]
        L.ccq_cuda_grouped.argtypes = [vp, i32, vp, vp, vp, C.c_int, vp, C.c_int, vp]
        L.ccq_cuda_experts_upload.argtypes = [vp, i32, C.c_int, C.POINTER(vp)]
        L.ccq_cuda_experts_matmul.argtypes = [vp, vp, vp, vp, C.c_int, vp, C.c_int, vp]
        L.ccq_cuda_moe_forward.argtypes = [vp, vp, vp, i64, i32, vp, C.c_int, vp, C.c_int, vp]
        L.ccq_cuda_search_codes.argtypes = [vp, i64, i32, i32, vp, i32, i32, i32, i32, vp, vp]
        L.ccq_quantize_host.argtypes = [vp, i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp]
        L.ccq_cuda_quantize_model.argtypes = [vp, i64, i64, i32, i32, i32, i32, vp]
        L.ccq_synthetic_packed.argtypes = [i64, i64, i32, i32, u64, vp, vp, vp, vp, vp]
        L.ccq_synthetic_matrix.argtypes = [i64, i64, i32, u64, vp]
        L.ccq_nccl_unique_id.argtypes = [vp]
        L.ccq_nccl_comm_init.argtypes = [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]
        L.ccq_nccl_comm_destroy.argtypes = [vp]
        L.ccq_cuda_shard_allgather.argtypes = [vp, i64, C.c_int, C.c_int, vp, C.c_int, i64, vp, C.c_int, i64,
                                               vp, vp]
        L.ccq_dequantize_host.argtypes = [vp, vp]
        L.ccq_gemv_host.argtypes = [vp, vp, u64, vp, u64]
        L.ccq_gemv_batch_host.argtypes = [vp, vp, i64, i64, vp, i64, i64]
        L.ccq_model_payload_bytes.argtypes = [vp, C.POINTER(u64)]
        L.ccq_group_geometry.argtypes = [i32, i32, vp]
        L.ccq_clustered_code_value.argtypes = [C.c_uint8, C.c_float, C.c_float, i32,
                                               C.POINTER(C.c_uint16)]
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != 0:
        msg = lib().ccq_cuda_last_error().decode(errors="replace")
        raise _STATUS.get(st, CcqError)(msg)


def launch_count() -> int:
    """Kernels launched by libccq_b200.so in this process."""
    return int(lib().ccq_cuda_launch_count())


def _np_ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data


@dataclass
class PackedModel:
    """ccq::PackedModel (container.hpp:37-52): the sections exactly as stored."""
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

    @staticmethod
    def from_sections(s) -> "PackedModel":
        return PackedModel(int(s.rows), int(s.cols), int(s.family), int(s.group_size),
                           np.ascontiguousarray(s.code_payload, np.uint8),
                           np.ascontiguousarray(s.scale_payload, np.uint8),
                           np.ascontiguousarray(s.super_scales, np.float32),
                           np.ascontiguousarray(s.cluster_scales, np.float32),
                           np.ascontiguousarray(s.cluster_zero_points, np.float32),
                           int(getattr(s, "rounds", 0)))

    def groups_per_row(self) -> int:
        return 0 if self.group_size == 0 else self.cols // self.group_size

    def group_count(self) -> int:
        return self.rows * self.groups_per_row()

    def _view(self) -> _View:
        arrs = [np.ascontiguousarray(self.code_payload, np.uint8),
                np.ascontiguousarray(self.scale_payload, np.uint8),
                np.ascontiguousarray(self.super_scales, np.float32),
                np.ascontiguousarray(self.cluster_scales, np.float32),
                np.ascontiguousarray(self.cluster_zero_points, np.float32)]
        v = _View(self.rows, self.cols, self.family, self.group_size, self.rounds, 0,
                  _np_ptr(arrs[0]), arrs[0].size, _np_ptr(arrs[1]), arrs[1].size,
                  _np_ptr(arrs[2]), arrs[2].size, _np_ptr(arrs[3]), arrs[3].size,
                  _np_ptr(arrs[4]), arrs[4].size)
        v._keep = arrs
        return v


def load_model(path: str) -> PackedModel:
    """ccq::load_model (container.cpp:428-432), host side."""
    v = _View()
    owner = C.c_void_p()
    _check(lib().ccq_container_open(path.encode(), C.byref(v), C.byref(owner)))
    try:
        def arr(ptr, n, dt):
            if not ptr or n == 0:
                return np.zeros(0, dt)
            nbytes = n * np.dtype(dt).itemsize
            return np.frombuffer(C.string_at(ptr, nbytes), dt).copy()
        return PackedModel(v.rows, v.cols, v.family, v.group_size,
                           arr(v.code_payload, v.code_bytes, np.uint8),
                           arr(v.scale_payload, v.scale_bytes, np.uint8),
                           arr(v.super_scales, v.n_super_scales, np.float32),
                           arr(v.cluster_scales, v.n_cluster_scales, np.float32),
                           arr(v.cluster_zero_points, v.n_cluster_zero_points, np.float32),
                           v.rounds)
    finally:
        lib().ccq_container_close(owner)


class DeviceModel:
    """A packed model resident in HBM (ccq_dev_model)."""

    def __init__(self, handle: C.c_void_p, host: PackedModel | None = None):
        self.h = handle
        info = ModelInfo()
        _check(lib().ccq_cuda_model_info(self.h, C.byref(info)))
        self.info = info
        self.rows, self.cols = info.rows, info.cols
        self.family, self.group_size = info.family, info.group_size
        self.device = info.device
        self.host = host

    @staticmethod
    def upload(model: PackedModel, device: int = 0, rows: tuple | None = None) -> "DeviceModel":
        h = C.c_void_p()
        v = model._view()
        if rows is None:
            _check(lib().ccq_cuda_model_upload(C.byref(v), device, C.byref(h)))
        else:
            _check(lib().ccq_cuda_model_upload_rows(C.byref(v), rows[0], rows[1], device,
                                                    C.byref(h)))
        return DeviceModel(h, model)

    @staticmethod
    def load(path: str, device: int = 0) -> "DeviceModel":
        h = C.c_void_p()
        _check(lib().ccq_cuda_model_load(path.encode(), device, C.byref(h)))
        return DeviceModel(h)

    @property
    def payload_bytes(self) -> int:
        out = C.c_uint64()
        _check(lib().ccq_model_payload_bytes(self.h, C.byref(out)))
        return int(out.value)

    def free(self) -> None:
        if getattr(self, "h", None):
            lib().ccq_cuda_model_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _dev(model) -> DeviceModel:
    if isinstance(model, DeviceModel):
        return model
    if isinstance(model, PackedModel):
        cache = getattr(model, "_dev_cache", None)
        if cache is None:
            cache = DeviceModel.upload(model)
            object.__setattr__(model, "_dev_cache", cache)
        return cache
    raise TypeError("expected PackedModel or DeviceModel")


# ---- reference-signature entry points (host buffers, synchronous) ----

def dequantize(model) -> np.ndarray:
    """ccq::dequantize (kernels.hpp:36): dense rows x cols f32, bit-exact."""
    d = _dev(model)
    out = np.empty((d.rows, d.cols), np.float32)
    _check(lib().ccq_dequantize_host(d.h, _np_ptr(out)))
    return out


def gemv(model, x, y=None) -> np.ndarray:
    """ccq::gemv (kernels.hpp:39)."""
    d = _dev(model)
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    out = np.empty(d.rows, np.float32) if y is None else y
    if not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous):
        raise ShapeError("y must be a C-contiguous float32 array")
    _check(lib().ccq_gemv_host(d.h, _np_ptr(x), x.size, _np_ptr(out), out.size))
    return out


def gemv_batch(model, x, y=None) -> np.ndarray:
    """ccq::gemv_batch (kernels.hpp:43): Y = X W^T."""
    d = _dev(model)
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != 2:
        raise ShapeError("gemv_batch expects a 2-D activation matrix")
    out = np.empty((x.shape[0], d.rows), np.float32) if y is None else y
    if not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous and out.ndim == 2):
        raise ShapeError("y must be a C-contiguous 2-D float32 array")
    _check(lib().ccq_gemv_batch_host(d.h, _np_ptr(x), x.shape[0], x.shape[1], _np_ptr(out),
                                     out.shape[0], out.shape[1]))
    return out


def model_payload_bytes(model) -> int:
    """ccq::model_payload_bytes (kernels.hpp:51)."""
    if isinstance(model, PackedModel):
        from math import ceil  # noqa: F401
        return int(model.code_payload.size + model.scale_payload.size + 4 * model.rows
                   + 4 * model.cluster_scales.size + 4 * model.cluster_zero_points.size)
    return _dev(model).payload_bytes


def group_geometry(family: int, group_size: int) -> dict:
    g = (C.c_int32 * 6)()
    _check(lib().ccq_group_geometry(family, group_size, g))
    keys = ("group_size", "full_words", "has_tail", "words_per_group", "embedded_scale",
            "payload_bytes")
    return dict(zip(keys, list(g)))


def clustered_code_value(q: int, alpha: float, beta: float, code_bits: int = 15) -> int:
    out = C.c_uint16()
    _check(lib().ccq_clustered_code_value(q, alpha, beta, code_bits, C.byref(out)))
    return out.value


# ---- device-resident layer (torch CUDA tensors) ----

def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


_DTYPE_CODES = None


def _torch_dtype_code(t) -> int:
    global _DTYPE_CODES
    if _DTYPE_CODES is None:
        import torch
        _DTYPE_CODES = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
    return _DTYPE_CODES[t.dtype]


def decode(model: DeviceModel, levels=None, weights=None, stream=None) -> None:
    """Kernel (a): levels (int8, state - zero_point) and/or f32 weights."""
    _check(lib().ccq_cuda_decode(model.h, None if levels is None else levels.data_ptr(),
                                 None if weights is None else weights.data_ptr(),
                                 _stream_ptr(stream)))


def matmul(model: DeviceModel, x, out=None, kernel: str = "auto", out_dtype=None, stream=None):
    """y[M, rows] = x[M, cols] . W^T on the device (kernels (b)/(c))."""
    import torch
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if not x.is_contiguous():
        raise ShapeError("activations must be contiguous")
    if x.shape[1] != model.cols:
        raise ShapeError("activation width does not match the model")
    if not x.is_cuda:
        raise ShapeError("activations must be a CUDA tensor")
    if out is None:
        out = torch.empty(x.shape[0], model.rows, dtype=out_dtype or torch.float32,
                          device=x.device)
    elif (tuple(out.shape) != (x.shape[0], model.rows) or out.dtype not in (torch.float32, torch.bfloat16)
          or not out.is_contiguous() or out.device != x.device):
        raise ShapeError("out must be a contiguous float32/bfloat16 [M, rows] tensor on the activations' device")
    L = lib()
    fn = L.ccq_cuda_matmul if kernel == "auto" else {"gemv": L.ccq_cuda_gemv, "gemm": L.ccq_cuda_gemm}[kernel]
    _check(fn(model.h, x.data_ptr(), _torch_dtype_code(x), x.shape[0], out.data_ptr(),
              _torch_dtype_code(out), _stream_ptr(stream)))
    return out


class Experts(DeviceModel):
    """E experts stacked in one device model (kernel (d), one launch)."""

    @staticmethod
    def upload(models, device: int = 0) -> "Experts":
        views = (_View * len(models))()
        keep = []
        for i, m in enumerate(models):
            v = m._view()
            keep.append(v)
            views[i] = v
        h = C.c_void_p()
        _check(lib().ccq_cuda_experts_upload(views, len(models), device, C.byref(h)))
        ex = Experts(h)
        ex.num_experts = len(models)
        ex.rows_per_expert = models[0].rows
        return ex


def experts_matmul(experts: "Experts", offsets, x, out=None, out_dtype=None, stream=None,
                   offsets_dev=None):
    """y[T, rows_per_expert] for expert-major tokens x[T, cols].

    `offsets` (E+1 host ints) sizes the launch; `offsets_dev` (the same values
    as a device int32 tensor) may be passed to skip the per-call upload."""
    import torch
    offs = np.ascontiguousarray(np.asarray(offsets, np.int32))
    if offs.size != experts.num_experts + 1:
        raise ShapeError("offsets must have num_experts+1 entries")
    if not x.is_contiguous() or x.dim() != 2 or x.shape[1] != experts.cols or x.shape[0] < offs[-1]:
        raise ShapeError("activations must be contiguous [offsets[-1], cols]")
    offs_dev = offsets_dev if offsets_dev is not None else torch.from_numpy(offs).to(x.device)
    if out is None:
        out = torch.empty(int(offs[-1]), experts.rows_per_expert, dtype=out_dtype or torch.float32,
                          device=x.device)
    _check(lib().ccq_cuda_experts_matmul(experts.h, offs_dev.data_ptr(), _np_ptr(offs), x.data_ptr(),
                                         _torch_dtype_code(x), out.data_ptr(), _torch_dtype_code(out),
                                         _stream_ptr(stream)))
    return out


def moe_forward(experts: "Experts", topk_ids, topk_weights, x, out=None, out_dtype=None, stream=None,
                validate: bool = True):
    """MoE layer with routing (ccq_cuda_moe_forward): x[T, cols] in token order,
    topk_ids / topk_weights [T, k] on the device -> y[T, rows_per_expert] =
    sum_j w[t, j] * expert_{ids[t, j]}(x[t]).

    The library call never synchronises (CUDA-graph capturable); with
    validate=True (default) the ids are range-checked here first (one host
    read), pass validate=False inside a captured serving loop."""
    import torch
    if validate and topk_ids.numel():
        lo, hi = int(topk_ids.min().item()), int(topk_ids.max().item())
        if lo < 0 or hi >= experts.num_experts:
            raise ShapeError(f"router expert id out of range [0, {experts.num_experts})")
    if topk_ids.dtype != torch.int32 or topk_weights.dtype != torch.float32:
        raise ShapeError("topk_ids must be int32 and topk_weights float32")
    if topk_ids.shape != topk_weights.shape or topk_ids.dim() != 2 or topk_ids.shape[0] != x.shape[0]:
        raise ShapeError("topk_ids / topk_weights must be [T, k] with T = x.shape[0]")
    if not (x.is_contiguous() and topk_ids.is_contiguous() and topk_weights.is_contiguous()):
        raise ShapeError("operands must be contiguous")
    if out is None:
        out = torch.empty(x.shape[0], experts.rows_per_expert, dtype=out_dtype or torch.float32,
                          device=x.device)
    _check(lib().ccq_cuda_moe_forward(experts.h, topk_ids.data_ptr(), topk_weights.data_ptr(), x.shape[0],
                                      topk_ids.shape[1], x.data_ptr(), _torch_dtype_code(x), out.data_ptr(),
                                      _torch_dtype_code(out), _stream_ptr(stream)))
    return out


# EncodingConfig (state_bits L, states_per_code N, transition_bits S) of each
# family's code parts (coding.cpp:24-27): 2.75, 2.06, and the 2.5 hybrid's two parts.
ENCODINGS = {"2.75": (4, 3, 2), "2.06": (6, 4, 3), "2.5-high": (3, 3, 2), "2.5-low": (3, 4, 2)}


def search_codes(targets, scales, config, zero_point=None, valid=None, stream=None):
    """Quantizer step on the GPU (ccq_cuda_search_codes): the reference's
    search_codes (quantizer.cpp:36-103) for every row of targets[n, >=valid]
    (f32, CUDA) with scales[n] (f64, CUDA) -> int32 codes[n], bit-identical.
    zero_point defaults to 2^(L-1) (the family schemes' zero point)."""
    import torch
    L, N, S = config
    if zero_point is None:
        zero_point = 1 << (L - 1)
    if targets.dim() != 2 or targets.dtype != torch.float32 or scales.dtype != torch.float64:
        raise ShapeError("targets must be [n, k] float32 and scales float64")
    if not (targets.is_contiguous() and scales.is_contiguous()) or scales.numel() != targets.shape[0]:
        raise ShapeError("targets / scales must be contiguous with one scale per row")
    valid = targets.shape[1] if valid is None else valid
    codes = torch.empty(targets.shape[0], dtype=torch.int32, device=targets.device)
    _check(lib().ccq_cuda_search_codes(targets.data_ptr(), targets.shape[0], valid, targets.shape[1],
                                       scales.data_ptr(), zero_point, L, N, S, codes.data_ptr(),
                                       _stream_ptr(stream)))
    return codes


def quantize(weights, family, group_size: int = 64, rounds: int = 2, device: int = 0) -> PackedModel:
    """pack_model(quantize_tensor(W)) with the search on the GPU
    (ccq_quantize_host): W[rows, cols] f32 (host) -> PackedModel whose
    sections are bit-identical to the reference quantizer's."""
    w = np.ascontiguousarray(weights, np.float32)
    if w.ndim != 2:
        raise ShapeError("weights must be a 2-D matrix")
    fam = FAMILIES[family] if isinstance(family, str) else int(family)
    rows, cols = w.shape
    geo = group_geometry(fam, group_size)
    groups = rows * (cols // group_size) if group_size > 0 else 0
    code = np.zeros(groups * geo["payload_bytes"], np.uint8)
    scale = np.zeros(0 if geo["embedded_scale"] else (groups + 1) // 2, np.uint8)
    sup = np.zeros(rows, np.float32)
    cl = fam == FAMILIES["2.06"]
    cs = np.zeros(rows if cl else 0, np.float32)
    czp = np.zeros(rows if cl else 0, np.float32)
    _check(lib().ccq_quantize_host(_np_ptr(w), rows, cols, fam, group_size, rounds, device, _np_ptr(code),
                                   _np_ptr(scale), _np_ptr(sup), _np_ptr(cs), _np_ptr(czp)))
    return PackedModel(rows, cols, fam, group_size, code, scale, sup, cs, czp, rounds)


def quantize_to_device(weights, family, group_size: int = 64, rounds: int = 2) -> DeviceModel:
    """Weights already on the GPU (torch f32 CUDA tensor [rows, cols]) ->
    quantized, packed and uploaded DeviceModel, no host round trip
    (ccq_cuda_quantize_model)."""
    if weights.dim() != 2 or not weights.is_cuda or not weights.is_contiguous():
        raise ShapeError("weights must be a contiguous 2-D CUDA tensor")
    import torch
    if weights.dtype != torch.float32:
        raise ShapeError("weights must be float32")
    fam = FAMILIES[family] if isinstance(family, str) else int(family)
    h = C.c_void_p()
    _check(lib().ccq_cuda_quantize_model(weights.data_ptr(), weights.shape[0], weights.shape[1], fam, group_size,
                                         rounds, weights.device.index or 0, C.byref(h)))
    return DeviceModel(h)


def grouped(models, offsets, x, out=None, out_dtype=None, stream=None):
    """Kernel (d): expert-major grouped matmul; offsets has E+1 entries."""
    import torch
    E = len(models)
    offs = np.ascontiguousarray(np.asarray(offsets, np.int32))
    if offs.size != E + 1:
        raise ShapeError("offsets must have len(models)+1 entries")
    handles = (C.c_void_p * E)(*[m.h for m in models])
    offs_dev = torch.from_numpy(offs).to(x.device)
    if out is None:
        out = torch.empty(int(offs[-1]), models[0].rows, dtype=out_dtype or torch.float32,
                          device=x.device)
    _check(lib().ccq_cuda_grouped(handles, E, offs_dev.data_ptr(), _np_ptr(offs), x.data_ptr(),
                                  _torch_dtype_code(x), out.data_ptr(), _torch_dtype_code(out),
                                  _stream_ptr(stream)))
    return out
