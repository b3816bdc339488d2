"""GPU exhaustive code search (ccq_cuda_search_codes, csrc/quantize.cu) against
the reference's own search_codes (quantizer.cpp:36-103, compiled from
/root/reference into oracle/_ref by oracle/Makefile): codes must be
bit-identical, including ties (smallest code wins) and short tails."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_err(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def _ref_codes(oracle, t, scales, valid, zp, cfg):
    L = oracle.ref()
    n, stride = t.shape
    out = np.zeros(n, np.uint32)
    st = L.ccqref_search_codes(t.ctypes.data, n, valid, stride, scales.ctypes.data, zp, cfg[0], cfg[1], cfg[2],
                               out.ctypes.data)
    assert st == 0, L.ccqref_last_error()
    return out


@pytest.mark.parametrize("name", ["2.75", "2.06", "2.5-high", "2.5-low"])
def test_search_codes_bit_exact(oracle, ccq, cuda, name):
    torch = cuda
    cfg = ccq.ENCODINGS[name]
    L, N, S = cfg
    zp = 1 << (L - 1)
    rng = np.random.default_rng(7 + L * 10 + N)
    n = 3000 if name != "2.06" else 600
    for valid in range(1, N + 1):
        t = (rng.standard_normal((n, N)) * rng.uniform(0.01, 2.0, (n, 1))).astype(np.float32)
        # scales as the quantizer seeds them (max |w| / (2^(L-1) - 1)) with jitter, plus edge rows
        sc = (np.abs(t[:, :valid]).max(axis=1) / float(zp - 1)) * rng.uniform(0.5, 1.5, n)
        t[:5] = 0.0          # all costs tie -> code 0
        sc[5:10] = 0.0       # scale 0: every state reconstructs 0 -> ties
        t[10:15] = np.float32(1e30)  # huge targets
        sc = np.ascontiguousarray(sc, np.float64)
        want = _ref_codes(oracle, t, sc, valid, zp, cfg)
        got = ccq.search_codes(torch.from_numpy(t).cuda(), torch.from_numpy(sc).cuda(), cfg, valid=valid)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().astype(np.uint32), want), (name, valid)


def test_search_codes_quantizer_shaped_targets(oracle, ccq, cuda):
    """Subvectors cut from Gaussian weight groups with the quantizer's initial
    scale (init_group_scale, quantizer.cpp:29-34): the 2.06 search that
    dominates quantize_tensor."""
    torch = cuda
    cfg = ccq.ENCODINGS["2.06"]
    rng = np.random.default_rng(11)
    w = rng.standard_normal((32, 64)).astype(np.float32) * 0.02
    scale = np.abs(w.astype(np.float64)).max(axis=1) / 31.0
    t = np.ascontiguousarray(w.reshape(-1, 4))
    sc = np.repeat(scale, 16).astype(np.float64)
    want = _ref_codes(oracle, t, sc, 4, 32, cfg)
    got = ccq.search_codes(torch.from_numpy(t).cuda(), torch.from_numpy(sc).cuda(), cfg)
    assert np.array_equal(got.cpu().numpy().astype(np.uint32), want)


def test_search_codes_errors(ccq, cuda):
    torch = cuda
    t = torch.zeros(4, 4, device="cuda")
    s = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ccq.ConfigError):
        ccq.search_codes(t, s, (4, 3, 5))   # S > L
    with pytest.raises(ccq.ConfigError):
        ccq.search_codes(t, s, (8, 4, 4))   # 20 bits > 16
    with pytest.raises(ccq.ShapeError):
        ccq.search_codes(t, s, (4, 3, 2))   # 4 values > N = 3
    with pytest.raises(ccq.ShapeError):
        ccq.search_codes(t, s, (4, 3, 2), valid=0)


def _sections_equal(a, b):
    assert a.rows == b.rows and a.cols == b.cols and a.family == b.family and a.group_size == b.group_size
    assert np.array_equal(np.asarray(a.code_payload, np.uint8), np.asarray(b.code_payload, np.uint8)), "codes"
    assert np.array_equal(np.asarray(a.scale_payload, np.uint8), np.asarray(b.scale_payload, np.uint8)), "scales"
    for x, y, what in ((a.super_scales, b.super_scales, "super"), (a.cluster_scales, b.cluster_scales, "cs"),
                       (a.cluster_zero_points, b.cluster_zero_points, "czp")):
        assert np.array_equal(np.asarray(x, np.float32).view(np.uint32), np.asarray(y, np.float32).view(np.uint32)), what


@pytest.mark.parametrize("fam,gs,rounds", [(0, 64, 2), (1, 64, 2), (2, 64, 2), (2, 64, 0), (0, 66, 1),
                                           (2, 65, 2), (1, 57, 3), (0, 64, 0)])
def test_gpu_quantizer_packed_sections_bit_exact(oracle, ccq, cuda, fam, gs, rounds):
    """ccq_quantize_host == the reference's pack_model(quantize_tensor(W))
    byte for byte (codes, side-band nibbles, super / cluster scales as f32
    bits), across families, tails and refinement rounds; plus rows that are
    all zero, constant and with one outlier."""
    rng = np.random.default_rng(fam * 100 + gs + rounds)
    rows, cols = 12, gs * 3
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    w[2, 5] = 3.0
    w[0] = 0.0
    if fam != 2:  # 2.06 rejects a constant row (next test)
        w[1] = 0.5
    want = oracle.RefModel.quantize(w, fam, gs, rounds, threads=1).sections()
    got = ccq.quantize(w, fam, gs, rounds)
    _sections_equal(got, want)
    # and the GPU decode of the GPU-quantized model equals the reference reconstruction
    d = ccq.DeviceModel.upload(got)
    assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(want).view(np.uint32))


def test_gpu_quantizer_layer_size(oracle, ccq, cuda):
    """A 256 x 4096 2.06 slab (4096 groups, 65,536 searches of 32,768 leaves
    per round) against the reference run on all host threads."""
    rng = np.random.default_rng(3)
    w = (rng.standard_normal((256, 4096)) * 0.02).astype(np.float32)
    want = oracle.RefModel.quantize(w, 2, 64, 1, threads=0).sections()
    got = ccq.quantize(w, 2, 64, 1)
    _sections_equal(got, want)


def test_gpu_quantizer_206_constant_row_domain_error(oracle, ccq, cuda):
    """A constant 2.06 row quantizes to one repeated high code word, which
    clusters to code_scale 1 at that zero point; the reference's
    build_cluster_table then raises DomainError (coding.hpp:145-148) - so must
    the GPU quantizer, same text."""
    rng = np.random.default_rng(5)
    w = (rng.standard_normal((3, 128)) * 0.02).astype(np.float32)
    w[1] = 0.25
    with pytest.raises(oracle.OracleError) as ref_err:
        oracle.RefModel.quantize(w, 2, 64, 2, threads=1)
    with pytest.raises(ccq.DomainError) as gpu_err:
        ccq.quantize(w, 2, 64, 2)
    assert str(ref_err.value).split("DomainError: ")[-1] in str(gpu_err.value)


@pytest.mark.parametrize("name,fam", [("2.06", 2), ("2.75", 0), ("2.5", 1)])
def test_cpp_api_quantize_matches_reference(oracle, ccq, cuda, tmp_path, name, fam):
    """The drop-in C++ API (ccq::cuda::quantize, tools/ccq_gpu_quantize.cpp)
    writes the reference quantizer's sections byte for byte."""
    import os
    import subprocess
    from conftest import ROOT
    lib_dir = os.path.join(ROOT, "paper_2507_07145_b200")
    exe = tmp_path / "ccq_gpu_quantize"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tools", "ccq_gpu_quantize.cpp"), "-o", str(exe),
                    os.path.join(lib_dir, "libccq_b200.so"), f"-Wl,-rpath,{lib_dir}"], check=True)
    w = (np.random.default_rng(fam).standard_normal((16, 256)) * 0.02).astype(np.float32)
    src, dst = tmp_path / "w.f32", tmp_path / "out.bin"
    w.tofile(src)
    r = subprocess.run([str(exe), str(src), "16", "256", name, "64", "2", str(dst)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    s = oracle.RefModel.quantize(w, fam, 64, 2, threads=1).sections()
    want = b"".join(np.ascontiguousarray(a).tobytes() for a in
                    (s.code_payload, s.scale_payload, s.super_scales, s.cluster_scales, s.cluster_zero_points))
    assert dst.read_bytes() == want


@pytest.mark.parametrize("fam", [2, 0, 1])
def test_quantize_to_device_model(oracle, ccq, cuda, fam):
    """Weights in HBM -> quantize -> device re-layout without a host round trip
    (ccq_cuda_quantize_model, device-resident views into the upload): the
    model decodes bit-identically to the reference quantizer's packed model
    and its matmul matches the oracle."""
    torch = cuda
    w = (np.random.default_rng(40 + fam).standard_normal((48, 512)) * 0.02).astype(np.float32)
    s = oracle.RefModel.quantize(w, fam, 64, 2, threads=1).sections()
    d = ccq.quantize_to_device(torch.from_numpy(w).cuda(), fam, 64, 2)
    assert d.rows == 48 and d.cols == 512
    assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(s).view(np.uint32))
    x = oracle.random_matrix(3, 512, "gaussian", 7)
    assert rel_err(ccq.gemv_batch(d, x), oracle.gemv_batch(s, x)) < 1e-3
