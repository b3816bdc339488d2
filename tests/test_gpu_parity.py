"""GPU parity: the sm_100a kernels against the CPU oracle on the same inputs.

Bar (BASELINE.json north_star): decoded levels and dequantized weights are
bit-exact; matmul outputs are within relative Frobenius error 1e-3 (fp32
accumulation vs the reference's double accumulation).  We assert a much
tighter REL_TOL so regressions show up long before the contract bound.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CONTRACT_TOL = 1e-3  # north_star: rel. err <= 1e-3
REL_TOL = 5e-5       # what the kernels achieve (fp32 accumulate; 2.5 is the loosest)


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.sqrt((want * want).sum())
    num = np.sqrt(((got - want) ** 2).sum())
    return num if den == 0 else num / den


def bf16_round(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


SHAPES = [(1, 64), (8, 128), (33, 192), (96, 128), (257, 4096), (130, 14336), (5, 2048 + 64)]


@pytest.fixture(scope="module")
def models(oracle, ccq, cuda):
    out = {}
    for fam in (0, 1, 2):
        for (rows, cols) in SHAPES:
            s = oracle.random_packed(rows, cols, fam, 64, seed=rows * 31 + cols + fam)
            out[(fam, rows, cols)] = (s, ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s)))
    return out


# ---------------------------------------------------------------- decode (a) --

@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES)
def test_decode_bit_exact(models, oracle, ccq, cuda, fam, shape):
    torch = cuda
    s, d = models[(fam, *shape)]
    lv = torch.empty(shape, dtype=torch.int8, device="cuda")
    w = torch.empty(shape, dtype=torch.float32, device="cuda")
    ccq.decode(d, levels=lv, weights=w)
    torch.cuda.synchronize()
    assert np.array_equal(lv.cpu().numpy(), oracle.levels(s))
    assert np.array_equal(w.cpu().numpy().view(np.uint32), oracle.dequantize(s).view(np.uint32))


@pytest.mark.parametrize("fam,gs", [(0, 66), (2, 65), (1, 57), (0, 64), (2, 64)])
def test_decode_non_default_geometry(oracle, ccq, cuda, fam, gs):
    torch = cuda
    s = oracle.random_packed(9, gs * 5, fam, gs, seed=gs + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    lv = torch.empty(9, gs * 5, dtype=torch.int8, device="cuda")
    w = torch.empty(9, gs * 5, dtype=torch.float32, device="cuda")
    ccq.decode(d, levels=lv, weights=w)
    assert np.array_equal(lv.cpu().numpy(), oracle.levels(s))
    assert np.array_equal(w.cpu().numpy().view(np.uint32), oracle.dequantize(s).view(np.uint32))
    # generic GEMV path for non-64 group sizes
    x = oracle.random_matrix(3, gs * 5, "gaussian", 4)
    y = ccq.gemv_batch(d, x)
    assert rel_err(y, oracle.gemv_batch(s, x)) < REL_TOL


@pytest.mark.parametrize("name", ["2.75", "2.5", "2.06"])
def test_acceptance_fixture_decode(oracle, ccq, cuda, name):
    """Criterion 6 on the GPU: the reference-written container decodes
    bit-identically to the reference's quantizer reconstruction."""
    import hashlib
    import json
    gold = json.load(open(os.path.join(GOLDEN, "golden.json")))["acceptance"][name]
    path = os.path.join(GOLDEN, f"acc512_{name}.ccq")
    d = ccq.DeviceModel.load(path)
    deq = ccq.dequantize(d)
    assert hashlib.sha256(deq.tobytes()).hexdigest() == gold["recon_sha"]
    ref = np.load(os.path.join(GOLDEN, f"acc512_{name}.npz"))
    y = ccq.gemv_batch(d, ref["x"])
    assert rel_err(y, ref["y"]) < REL_TOL


def test_dequantize_host_matches_oracle(models, oracle, ccq):
    for fam in (0, 1, 2):
        s, d = models[(fam, 257, 4096)]
        assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(s).view(np.uint32))


def test_zero_scale_codes_decode_to_zero(oracle, ccq, cuda):
    # test_kernels.cpp:89-101
    for fam in (0, 1, 2):
        s = oracle.random_packed(4, 128, fam, 64, 21)
        if fam == 2:
            s.scale_payload[:] = 0
        else:
            codes = s.code_payload.reshape(-1, 22 if fam == 0 else 20)
            if fam == 0:
                codes[:, 21] &= 0xF0
            else:
                codes[:, 18] = 0
                codes[:, 19] &= 0xE0
        d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
        assert (ccq.dequantize(d) == 0).all()
        assert (ccq.gemv_batch(d, oracle.random_matrix(2, 128, "gaussian", 1)) == 0).all()


# ------------------------------------------------------------------ gemv (b) --

@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("M", [1, 2, 3, 4, 5])
def test_gemv_f32_matches_oracle(models, oracle, ccq, cuda, fam, shape, M):
    s, d = models[(fam, *shape)]
    x = oracle.random_matrix(M, shape[1], "gaussian", 1000 + M)
    y = ccq.gemv_batch(d, x)
    want = oracle.gemv_batch(s, x, threads=8)
    err = rel_err(y, want)
    assert err < REL_TOL, err
    assert err < CONTRACT_TOL


@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("M", [1, 2, 4, 8, 16])
def test_gemv_bf16_device(models, oracle, ccq, cuda, fam, M):
    torch = cuda
    s, d = models[(fam, 130, 14336)]
    x = oracle.random_matrix(M, 14336, "gaussian", 7 + M)
    xb = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xb, kernel="gemv")
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, bf16_round(x), threads=8)  # oracle fed the same bf16 x
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("M", [1, 3, 8, 9, 16, 21])
def test_gemv_tensor_pipe_bf16_all_shapes(models, oracle, ccq, cuda, fam, shape, M, monkeypatch):
    """The mma.sync GEMV (bf16 activations): every family, ragged rows/cols,
    token counts across the n8 / n16 tiles and the 16-token launch chunks
    (CCQ_FORCE_MMA routes M = 1 to it as well)."""
    monkeypatch.setenv("CCQ_FORCE_MMA", "1")
    torch = cuda
    s, d = models[(fam, *shape)]
    x = bf16_round(oracle.random_matrix(M, shape[1], "gaussian", 31 + M))
    xb = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xb, kernel="gemv")
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, x, threads=8)
    err = rel_err(y.cpu().numpy(), want)
    assert err < REL_TOL, err


@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("scale", [1e-30, 1e-6, 1.0, 3e4, 1e30])
def test_gemv_tensor_pipe_activation_range(models, oracle, ccq, cuda, fam, scale, monkeypatch):
    """Per-token power-of-two rescaling keeps f16 operands exact across the
    whole bf16 range; tokens of very different magnitude share one launch."""
    monkeypatch.setenv("CCQ_FORCE_MMA", "1")
    torch = cuda
    s, d = models[(fam, 257, 4096)]
    x = oracle.random_matrix(3, 4096, "gaussian", 5)
    x[1] *= scale
    x[2] *= 1.0 / scale if scale != 1.0 else 7.0
    x = bf16_round(x)
    y = ccq.matmul(d, torch.from_numpy(x).to("cuda").to(torch.bfloat16), kernel="gemv")
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, x, threads=8)
    got = y.cpu().numpy()
    for n in range(3):
        assert rel_err(got[n], want[n]) < REL_TOL, (n, rel_err(got[n], want[n]))


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_gemv_tensor_pipe_f16_in_bf16_out(models, oracle, ccq, cuda, fam):
    torch = cuda
    s, d = models[(fam, 130, 14336)]
    x = oracle.random_matrix(4, 14336, "gaussian", 9)
    xh = torch.from_numpy(x).to("cuda").to(torch.float16)
    y = ccq.matmul(d, xh, kernel="gemv", out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, xh.float().cpu().numpy(), threads=8)
    assert rel_err(y.float().cpu().numpy(), want) < 5e-3  # bf16 output rounding


def test_gemv_single_vector_and_shape_errors(models, oracle, ccq):
    s, d = models[(0, 33, 192)]
    x = oracle.random_matrix(1, 192, "uniform", 99)[0]
    assert rel_err(ccq.gemv(d, x), oracle.gemv_batch(s, x)[0]) < REL_TOL
    # test_kernels.cpp:151-161
    with pytest.raises(ccq.ShapeError):
        ccq.gemv(d, np.zeros(191, np.float32))
    with pytest.raises(ccq.ShapeError):
        ccq.gemv(d, np.zeros(192, np.float32), np.zeros(32, np.float32))
    with pytest.raises(ccq.ShapeError):
        ccq.gemv_batch(d, np.zeros((2, 192), np.float32), np.zeros((3, 33), np.float32))
    with pytest.raises(ccq.ShapeError):
        ccq.gemv_batch(d, np.zeros((2, 192), np.float32), np.zeros((2, 34), np.float32))


def test_gemv_zero_vector_and_linearity(models, oracle, ccq):
    # test_kernels.cpp:117-137
    s, d = models[(1, 96, 128)]
    assert (ccq.gemv(d, np.zeros(128, np.float32)) == 0).all()
    a = oracle.random_matrix(1, 128, "gaussian", 1)[0]
    b = oracle.random_matrix(1, 128, "gaussian", 2)[0]
    ya, yb, yab = ccq.gemv(d, a), ccq.gemv(d, b), ccq.gemv(d, 2 * a + b)
    assert rel_err(yab, 2 * ya + yb) < REL_TOL


def test_widening_domain_error_on_upload(oracle, ccq, cuda):
    """A stored byte whose widened code leaves [0, 2^15) raises DomainError
    (the reference raises the same error when decoding it, coding.hpp:145)."""
    s = oracle.random_packed(4, 128, 2, 64, 3)
    s.cluster_scales[1] = np.float32(200.0)
    s.cluster_zero_points[1] = np.float32(0.0)
    s.code_payload[32 * 1 + 5] = 255  # row 1 (32 bytes per row) gets q = 255 -> 51000
    with pytest.raises(ccq.DomainError):
        ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    # the same parameters are accepted when no such byte is stored
    s.code_payload[32:64] = np.minimum(s.code_payload[32:64], 100)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(s).view(np.uint32))


def test_widening_plans_exhaustive_random_rows(oracle, ccq, cuda):
    """Every q of many random (alpha, beta) rows, including tiny/huge alpha and
    exact-tie values, widens exactly as lround(q*alpha+beta)."""
    rng = np.random.default_rng(1)
    rows = 512
    s = oracle.random_packed(rows, 1024, 2, 64, 5)  # 16 groups x 16 B = 256 bytes per row
    alphas = np.concatenate([1 + rng.random(rows - 8) * 64, [2.5, 0.5, 1.0, 0.25, 1e-3, 127.9, 128.49, 3.0]])
    s.cluster_scales[:] = alphas.astype(np.float32)
    for r in range(rows):
        a = float(s.cluster_scales[r])
        s.cluster_zero_points[r] = np.float32(rng.random() * max(0.0, 32767 - 255 * a - 1))
    s.cluster_zero_points[-8:] = np.float32([0.5, 0.25, 7.0, 0.0, 3.5, 0.0, 0.0, 1.5])
    # every q appears in every row: bytes 0..255 (rows are 256 bytes wide)
    s.code_payload[:] = np.tile(np.arange(256, dtype=np.uint8), rows)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(s).view(np.uint32))


def test_row_sharded_upload_concatenates(oracle, ccq, cuda):
    s = oracle.random_packed(64, 512, 2, 64, 8)
    pm = ccq.PackedModel.from_sections(s)
    x = oracle.random_matrix(2, 512, "gaussian", 3)
    parts = [ccq.DeviceModel.upload(pm, rows=(r, r + 16)) for r in range(0, 64, 16)]
    y = np.concatenate([ccq.gemv_batch(p, x) for p in parts], axis=1)
    assert rel_err(y, oracle.gemv_batch(s, x)) < REL_TOL
    deq = np.concatenate([ccq.dequantize(p) for p in parts], axis=0)
    assert np.array_equal(deq.view(np.uint32), oracle.dequantize(s).view(np.uint32))


def test_empty_inputs(oracle, ccq, cuda):
    s = oracle.random_packed(0, 128, 0, 64, 1)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    assert ccq.dequantize(d).shape == (0, 128)
    s = oracle.random_packed(4, 128, 1, 64, 1)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    assert ccq.gemv_batch(d, np.zeros((0, 128), np.float32)).shape == (0, 4)


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_baseline_shape_full_size(oracle, ccq, cuda, fam):
    """BASELINE config 2 shape (d_in 4096 -> d_out 14336) at full size, M=1,
    against the (multithreaded) oracle."""
    s = oracle.random_packed(14336, 4096, fam, 64, seed=4096 * 31 + 14336)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(1, 4096, "gaussian", 4096 + 1)
    y = ccq.gemv_batch(d, x)
    assert rel_err(y, oracle.gemv_batch(s, x, threads=8)) < REL_TOL


# ------------------------------------------------------------ gemm (c) tcgen05 --

@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("shape", [(128, 512), (200, 4096), (384, 2048 + 64), (130, 14336), (64, 192),
                                   (1000, 8192 + 512)])
@pytest.mark.parametrize("M", [9, 32, 64, 100, 128, 256, 300])
def test_gemm_tcgen05_bf16(oracle, ccq, cuda, fam, shape, M):
    """All three families on tcgen05: exact f16 weight operands (2.5 as two
    exact parts with two TMEM accumulators), f32 accumulation."""
    torch = cuda
    rows, cols = shape
    s = oracle.random_packed(rows, cols, fam, 64, seed=rows + cols + M + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(M, cols, "gaussian", 17 + M)
    xb = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xb, kernel="gemm")
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, bf16_round(x), threads=8)
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_gemm_tcgen05_f32_input_within_contract(oracle, ccq, cuda, fam):
    s = oracle.random_packed(256, 1024, fam, 64, seed=3)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(64, 1024, "gaussian", 5)
    y = ccq.gemv_batch(d, x)  # M = 64 dispatches to the tcgen05 GEMM
    # f32 activations run as hi/lo f16 pairs: full f32-level accuracy
    assert rel_err(y, oracle.gemv_batch(s, x, threads=8)) < REL_TOL


@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("M", [1, 3, 31, 33, 200])
@pytest.mark.parametrize("scale", [1.0, 1e-6, 3e5])
def test_gemm_f32_input_scaling(oracle, ccq, cuda, fam, M, scale):
    """Per-token power-of-two scaling: tiny and huge activations stay exact."""
    torch = cuda
    s = oracle.random_packed(160, 1024, fam, 64, seed=M + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = (oracle.random_matrix(M, 1024, "gaussian", 40 + M) * np.float32(scale)).astype(np.float32)
    y = ccq.matmul(d, torch.from_numpy(x).cuda(), kernel="gemm")
    assert rel_err(y.cpu().numpy(), oracle.gemv_batch(s, x, threads=8)) < REL_TOL


@pytest.mark.parametrize("fam", [0, 1, 2])
def test_gemm_bf16_output(oracle, ccq, cuda, fam):
    torch = cuda
    s = oracle.random_packed(256, 1024, fam, 64, seed=4)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(48, 1024, "gaussian", 6)
    xb = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xb, kernel="gemm", out_dtype=torch.bfloat16)
    want = oracle.gemv_batch(s, bf16_round(x), threads=8)
    assert rel_err(y.float().cpu().numpy(), want) < 4e-3  # bf16 output rounding


@pytest.mark.parametrize("rows", [32768, 127 * 256 + 100, 127 * 256 + 200])
@pytest.mark.parametrize("M,xdt", [(150, "bf16"), (120, "bf16"), (70, "f32")])
def test_gemm_two_row_tile_ctas_by_default(oracle, ccq, cuda, rows, M, xdt):
    """Dense grids that fill >= 0.8 waves with 256-row CTAs take the two-row-
    tile GEMM by default (2.06, 128/160-column tiles, gemm_sm100.cu RT = 2),
    including a last CTA whose second 128-row box is absent (rows % 256 = 100)
    or partial (200)."""
    torch = cuda
    cols = 512
    s = oracle.random_packed(rows, cols, 2, 64, seed=rows + M)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(M, cols, "gaussian", 31 + M)
    if xdt == "bf16":
        xt = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
        x = bf16_round(x)
    else:
        xt = torch.from_numpy(x).to("cuda")
    y = ccq.matmul(d, xt, kernel="gemm")
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, x, threads=8)
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


# ------------------------------------------------------- grouped experts (d) --

def _expert_case(oracle, fam, E, rows, cols, counts, seed):
    secs = [oracle.random_packed(rows, cols, fam, 64, seed=seed * 97 + e) for e in range(E)]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    x = oracle.random_matrix(int(offs[-1]), cols, "gaussian", seed + 5) if offs[-1] else \
        np.zeros((0, cols), np.float32)
    want = np.zeros((int(offs[-1]), rows), np.float32)
    for e in range(E):
        if counts[e]:
            want[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], x[offs[e]:offs[e + 1]], threads=8)
    return secs, offs, x, want


@pytest.mark.parametrize("fam", [0, 1, 2])
@pytest.mark.parametrize("counts", [[5, 0, 70, 1], [0, 0, 0, 3], [130, 64, 0, 257], [1, 1, 1, 1]])
def test_experts_single_launch_matches_per_expert_oracle(oracle, ccq, cuda, fam, counts):
    torch = cuda
    E, rows, cols = len(counts), 200, 512
    secs, offs, x, want = _expert_case(oracle, fam, E, rows, cols, counts, seed=sum(counts) + fam)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s) for s in secs])
    xb = torch.from_numpy(bf16_round(x)).cuda().to(torch.bfloat16)
    wantb = np.zeros_like(want)
    for e in range(E):
        if counts[e]:
            wantb[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], bf16_round(x[offs[e]:offs[e + 1]]), threads=8)
    y = ccq.experts_matmul(ex, offs, xb)
    assert rel_err(y.cpu().numpy(), wantb) < REL_TOL
    y32 = ccq.experts_matmul(ex, offs, torch.from_numpy(x).cuda())
    assert rel_err(y32.cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("rows", [100, 128, 300, 512])
def test_experts_two_row_tile_ctas(oracle, ccq, cuda, rows):
    """Grouped 2.06 launches use 256-row CTAs (RT = 2): expert row counts whose
    last CTA has no second 128-row box (100, 300), exactly one box (128) or
    two full boxes (512)."""
    torch = cuda
    counts = [150, 40, 0, 97]
    E, cols = len(counts), 512
    secs, offs, x, _ = _expert_case(oracle, 2, E, rows, cols, counts, seed=rows)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s) for s in secs])
    xb = torch.from_numpy(bf16_round(x)).cuda().to(torch.bfloat16)
    want = np.zeros((int(offs[-1]), rows), np.float32)
    for e in range(E):
        if counts[e]:
            want[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], bf16_round(x[offs[e]:offs[e + 1]]), threads=8)
    y = ccq.experts_matmul(ex, offs, xb)
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("counts", [[1, 0, 0, 1, 0, 1, 1, 0], [0, 0, 3, 0, 0, 0, 0, 0], [2, 2, 2, 2, 2, 2, 2, 2],
                                    [1] * 8, [0, 16, 0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 1],
                                    [9, 16, 0, 12, 5, 1, 0, 16]])
@pytest.mark.parametrize("xdt", ["bf16", "f16"])
@pytest.mark.parametrize("fam,path", [(2, "rec"), (2, "box"), (0, "box"), (1, "box")])
def test_experts_decode_grouped_gemv(oracle, ccq, cuda, counts, xdt, fam, path, monkeypatch):
    """Decode batches (<= 16 routed rows per expert window): one tensor-pipe
    GEMV launch over the tiles of the experts that have tokens; experts without
    tokens are skipped.  2.06 on the record kernel and on the TMA-box kernel
    (CCQ_NO_REC), 2.75 / 2.5 on the TMA-box kernel."""
    torch = cuda
    monkeypatch.setenv("CCQ_NO_GROUPED_STREAM", "1")  # one-token batches would take the streaming kernel
    if path == "box":
        monkeypatch.setenv("CCQ_NO_REC", "1")
    E, rows, cols = 8, 48, 1024 + 64
    secs, offs, x, want = _expert_case(oracle, fam, E, rows, cols, counts, seed=sum(counts) * 3 + 1 + fam)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s_) for s_ in secs])
    tdt = torch.bfloat16 if xdt == "bf16" else torch.float16
    xt = torch.from_numpy(x).to("cuda").to(tdt)
    y = ccq.experts_matmul(ex, offs, xt)
    torch.cuda.synchronize()
    want = np.zeros((int(offs[-1]), rows), np.float32)
    xr = xt.float().cpu().numpy()
    for e in range(E):
        if counts[e]:
            want[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], xr[offs[e]:offs[e + 1]], threads=8)
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


def test_experts_one_launch_and_untouched_padding(oracle, ccq, cuda):
    torch = cuda
    counts = [3, 0, 40, 0, 9, 0, 0, 100]
    secs, offs, x, want = _expert_case(oracle, 2, 8, 256, 1024, counts, seed=11)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s) for s in secs])
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y = torch.full((int(offs[-1]) + 1, 256), 7.0, device="cuda")
    torch.cuda.synchronize()
    n0 = ccq.launch_count()
    ccq.experts_matmul(ex, offs, xb, out=y)
    torch.cuda.synchronize()
    assert ccq.launch_count() - n0 == 2  # activation pre-pass + one grouped GEMM
    assert (y[-1] == 7.0).all()
    wantb = np.zeros_like(want)
    for e in range(8):
        if counts[e]:
            wantb[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], bf16_round(x[offs[e]:offs[e + 1]]), threads=8)
    assert rel_err(y[:-1].cpu().numpy(), wantb) < REL_TOL


def test_experts_match_list_api(oracle, ccq, cuda):
    torch = cuda
    counts = [17, 2, 0, 33]
    secs, offs, x, want = _expert_case(oracle, 2, 4, 128, 256, counts, seed=2)
    pms = [ccq.PackedModel.from_sections(s) for s in secs]
    ex = ccq.Experts.upload(pms)
    ds = [ccq.DeviceModel.upload(p) for p in pms]
    xt = torch.from_numpy(x).cuda()
    a = ccq.experts_matmul(ex, offs, xt).cpu().numpy()
    b = ccq.grouped(ds, offs, xt).cpu().numpy()
    assert rel_err(a, want) < REL_TOL and rel_err(b, want) < REL_TOL


def test_experts_shape_errors(oracle, ccq, cuda):
    s0 = oracle.random_packed(64, 128, 2, 64, seed=1)
    s1 = oracle.random_packed(64, 192, 2, 64, seed=2)
    with pytest.raises(ccq.ShapeError):
        ccq.Experts.upload([ccq.PackedModel.from_sections(s0), ccq.PackedModel.from_sections(s1)])


# ------------------------------------------- BASELINE full sizes (sampled) --

def _slice_rows(oracle, sec, r0, r1):
    """Rows [r0, r1) of packed sections (the reference's group-major layout)."""
    g = oracle.group_geometry(sec.family, sec.group_size)
    gpr = sec.cols // sec.group_size
    pb = g["payload_bytes"]
    code = sec.code_payload[r0 * gpr * pb: r1 * gpr * pb].copy()
    if g["embedded_scale"]:
        scale = np.zeros(0, np.uint8)
    else:
        nib = np.array([(sec.scale_payload[i // 2] >> (4 * (i % 2))) & 0xF
                        for i in range(r0 * gpr, r1 * gpr)], np.uint16)
        scale = np.frombuffer(oracle.pack_cluster_scales(nib), np.uint8).copy()
    cs = sec.cluster_scales[r0:r1] if sec.cluster_scales.size else sec.cluster_scales
    czp = sec.cluster_zero_points[r0:r1] if sec.cluster_zero_points.size else sec.cluster_zero_points
    return oracle.Sections(r1 - r0, sec.cols, sec.family, sec.group_size, code, scale,
                           sec.super_scales[r0:r1].copy(), cs.copy(), czp.copy())


@pytest.mark.parametrize("fam", [2, 0, 1])
def test_prefill_config4_full_size_sampled(oracle, ccq, cuda, fam):
    """BASELINE configs[4] at full size (8192 -> 28672, M = 4096 tokens) on the
    tcgen05 GEMM: a 64-row sample of the output checked against the oracle
    on ALL tokens (2 x 64 x 8192 x 4096 flop on the CPU), plus linearity of
    the whole product in x."""
    torch = cuda
    s = oracle.random_packed(28672, 8192, fam, 64, seed=8192 * 31 + 28672 + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = bf16_round(oracle.random_matrix(4096, 8192, "gaussian", 4097))
    xt = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xt)
    torch.cuda.synchronize()
    rows = [(0, 32), (17000, 17032)]
    for r0, r1 in rows:
        want = oracle.gemv_batch(_slice_rows(oracle, s, r0, r1), x, threads=8)
        assert rel_err(y[:, r0:r1].cpu().numpy(), want) < REL_TOL
    # linearity: W(x1 + x2) == W x1 + W x2 (f32 accumulation tolerance)
    x2 = torch.from_numpy(bf16_round(oracle.random_matrix(4096, 8192, "gaussian", 4098))).to("cuda").to(torch.bfloat16)
    xs = (xt.float() + x2.float()).to(torch.bfloat16)
    lhs = ccq.matmul(d, xs)
    rhs = y + ccq.matmul(d, x2)
    exact = (xt.float() + x2.float() - xs.float()).abs().max().item() == 0.0
    tol = REL_TOL if exact else 1e-2  # bf16 rounding of the sum when not exact
    assert rel_err(lhs.cpu().numpy(), rhs.cpu().numpy()) < tol


@pytest.mark.parametrize("fam", [2, 0, 1])
def test_config4_shape_decode_batches_full_size(oracle, ccq, cuda, fam):
    """configs[4]'s 8192 -> 28672 layer at decode batches M = 1..8 on the
    tensor-pipe GEMV (kernel="gemv") and the auto dispatch: sampled rows
    against the oracle, and the WHOLE output against the tcgen05 GEMM (every
    row tile of every CTA; the record kernel's ring depth changes with M -
    S = 2 once aliased a stale stage at M = 6)."""
    torch = cuda
    s = oracle.random_packed(28672, 8192, fam, 64, seed=28672 + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    for M in range(1, 9):
        x = bf16_round(oracle.random_matrix(M, 8192, "gaussian", 100 + M))
        xt = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
        ref = ccq.matmul(d, xt, kernel="gemm")
        for kernel in ("gemv", "auto"):
            y = ccq.matmul(d, xt, kernel=kernel)
            torch.cuda.synchronize()
            assert rel_err(y.cpu().numpy(), ref.cpu().numpy()) < REL_TOL, (M, kernel)
            for r0, r1 in ((0, 16), (28656, 28672)):
                want = oracle.gemv_batch(_slice_rows(oracle, s, r0, r1), x, threads=8)
                assert rel_err(y[:, r0:r1].cpu().numpy(), want) < REL_TOL, (M, kernel, r0)


@pytest.mark.parametrize("name,E,din,dout,B", [("ERNIE", 64, 8192, 3584, 1), ("ERNIE", 64, 8192, 3584, 64),
                                               ("DeepSeek", 256, 7168, 2048, 1), ("DeepSeek", 256, 7168, 2048, 16),
                                               ("ERNIE", 64, 8192, 3584, 4096), ("DeepSeek", 256, 7168, 2048, 4096)])
def test_moe_configs_full_size_sampled(oracle, ccq, cuda, name, E, din, dout, B):
    """BASELINE configs[2]/[3] at full expert count and shape, top-8 routing,
    decode batches and the T = 4096-token prefill (32,768 routed pairs on the
    grouped tcgen05 GEMM): routed experts' output rows checked against the
    oracle (B = 4096: three experts, 48 of their tokens each - the CPU
    oracle is f64)."""
    torch = cuda
    rng = np.random.default_rng(B + E)
    counts = np.zeros(E, np.int64)
    for _ in range(B):
        counts[rng.choice(E, 8, replace=False)] += 1
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    secs = [oracle.random_packed(dout, din, 2, 64, seed=e + 7) for e in range(E)]
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(t) for t in secs])
    x = bf16_round(oracle.random_matrix(int(offs[-1]), din, "gaussian", 11))
    y = ccq.experts_matmul(ex, offs, torch.from_numpy(x).to("cuda").to(torch.bfloat16)).cpu().numpy()
    hit = [e for e in range(E) if counts[e]]
    sample = hit[:8] if B < 4096 else [hit[0], hit[len(hit) // 2], hit[-1]]
    for e in sample:
        t1 = offs[e + 1] if B < 4096 else min(offs[e + 1], offs[e] + 48)
        want = oracle.gemv_batch(secs[e], x[offs[e]:t1], threads=8)
        assert rel_err(y[offs[e]:t1], want) < REL_TOL, (name, e)


# ----------------------------------------------------------- randomized sweep --

@pytest.mark.parametrize("seed", list(range(64)))
def test_randomized_shapes_all_paths(oracle, ccq, cuda, seed):
    """Seeded random (family, rows, cols, M, dtypes, kernel) cases through the
    public dispatcher and the forced paths, each against the oracle."""
    torch = cuda
    rng = np.random.default_rng(1000 + seed)
    fam = int(rng.integers(0, 3))
    rows = int(rng.integers(1, 700))
    cols = 64 * int(rng.integers(1, 80))
    M = int(rng.choice([1, 2, 3, 5, 8, 9, 16, 17, 40, 100, 300]))
    kern = str(rng.choice(["auto", "gemv", "gemm"]))
    xdt = [torch.bfloat16, torch.float16, torch.float32][int(rng.integers(0, 3))]
    ydt = [torch.float32, torch.bfloat16][int(rng.integers(0, 2))]
    s = oracle.random_packed(rows, cols, fam, 64, seed=seed * 7 + 3)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = oracle.random_matrix(M, cols, "gaussian", seed)
    xt = torch.from_numpy(x).to("cuda").to(xdt)
    y = ccq.matmul(d, xt, kernel=kern, out_dtype=ydt)
    torch.cuda.synchronize()
    want = oracle.gemv_batch(s, xt.float().cpu().numpy(), threads=8)
    tol = REL_TOL if ydt == torch.float32 else 5e-3
    assert rel_err(y.float().cpu().numpy(), want) < tol, (fam, rows, cols, M, kern, xdt, ydt)


# ------------------------------------------------ MoE routing (permute/combine) --

@pytest.mark.parametrize("fam", [2, 0, 1])
@pytest.mark.parametrize("T,k,E", [(1, 8, 16), (5, 2, 6), (40, 8, 16), (300, 4, 8)])
def test_moe_forward_routing(oracle, ccq, cuda, fam, T, k, E):
    """Token-order x + router top-k -> weighted sum of the experts' outputs,
    against the oracle composition y[t] = sum_j w[t,j] * gemv(expert e(t,j), x[t])."""
    torch = cuda
    rows, cols = 48, 512
    rng = np.random.default_rng(T * 31 + k + fam)
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
    w = rng.random((T, k)).astype(np.float32)
    secs = [oracle.random_packed(rows, cols, fam, 64, seed=e + 50 * fam) for e in range(E)]
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(t) for t in secs])
    x = bf16_round(oracle.random_matrix(T, cols, "gaussian", T))
    y = ccq.moe_forward(ex, torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(),
                        torch.from_numpy(x).cuda().to(torch.bfloat16))
    torch.cuda.synchronize()
    want = np.zeros((T, rows), np.float64)
    for e in range(E):
        tok, slot = np.nonzero(ids == e)
        if tok.size:
            ye = oracle.gemv_batch(secs[e], x[tok], threads=8)
            for i in range(tok.size):
                want[tok[i]] += float(w[tok[i], slot[i]]) * ye[i]
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("fam", [2, 0])
def test_moe_forward_graph_capture_and_replay(oracle, ccq, cuda, fam):
    """ccq_cuda_moe_forward never synchronises: it is captured once in a CUDA
    graph and replayed with NEW routing and activations written into the
    captured input buffers; every replay matches the oracle composition
    (decode batch T = 4 and a prefill-sized batch T = 300, top-4 of 16)."""
    torch = cuda
    rows, cols, E, k = 64, 512, 16, 4
    secs = [oracle.random_packed(rows, cols, fam, 64, seed=e + 900 + fam) for e in range(E)]
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(t) for t in secs])
    for T in (4, 300):
        ids_d = torch.zeros(T, k, dtype=torch.int32, device="cuda")
        w_d = torch.zeros(T, k, dtype=torch.float32, device="cuda")
        x_d = torch.zeros(T, cols, dtype=torch.bfloat16, device="cuda")
        y_d = torch.empty(T, rows, dtype=torch.float32, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):  # warm-up (allocations, attributes) outside capture
            ccq.moe_forward(ex, ids_d, w_d, x_d, out=y_d, stream=s, validate=False)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ccq.moe_forward(ex, ids_d, w_d, x_d, out=y_d, stream=s, validate=False)
        for rep in range(3):
            rng = np.random.default_rng(T * 7 + rep + fam)
            ids = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
            w = rng.random((T, k)).astype(np.float32)
            x = bf16_round(oracle.random_matrix(T, cols, "gaussian", T + rep))
            ids_d.copy_(torch.from_numpy(ids))
            w_d.copy_(torch.from_numpy(w))
            x_d.copy_(torch.from_numpy(x).to(torch.bfloat16))
            g.replay()
            torch.cuda.synchronize()
            want = np.zeros((T, rows), np.float64)
            for e in range(E):
                tok, slot = np.nonzero(ids == e)
                if tok.size:
                    ye = oracle.gemv_batch(secs[e], x[tok], threads=8)
                    for i in range(tok.size):
                        want[tok[i]] += float(w[tok[i], slot[i]]) * ye[i]
            assert rel_err(y_d.cpu().numpy(), want) < REL_TOL, (T, rep)


def test_moe_forward_rejects_bad_expert_ids(ccq, cuda):
    torch = cuda
    from paper_2507_07145_b200.synthetic import random_packed
    ex = ccq.Experts.upload([random_packed(32, 256, 2, 64, e) for e in range(4)])
    ids = torch.tensor([[0, 7]], dtype=torch.int32, device="cuda")
    w = torch.ones(1, 2, device="cuda")
    with pytest.raises(ccq.ShapeError):
        ccq.moe_forward(ex, ids, w, torch.randn(1, 256, device="cuda").to(torch.bfloat16))


@pytest.mark.parametrize("fam,gs", [(2, 64), (0, 64), (1, 64), (2, 65), (0, 66), (1, 57)])
def test_device_loader_row_ranges_bit_exact(oracle, ccq, cuda, fam, gs):
    """The device-side loader (model.cu relayout_records/build_plans) for row
    ranges that start on odd group indices (odd groups per row, odd r0:
    side-band nibbles straddle bytes) and ranges ending inside a 16-row pad:
    each range decodes bit-identically to the oracle's rows."""
    torch = cuda
    rows, gpr = 45, 7  # odd groups per row; 7 groups < one 32-group chunk
    s = oracle.random_packed(rows, gs * gpr, fam, gs, seed=77 + fam + gs)
    pm = ccq.PackedModel.from_sections(s)
    lv_all = oracle.levels(s)
    w_all = oracle.dequantize(s)
    for r0, r1 in ((0, rows), (1, 2), (3, 20), (17, 45), (44, 45)):
        d = ccq.DeviceModel.upload(pm, rows=(r0, r1))
        lv = torch.empty(r1 - r0, gs * gpr, dtype=torch.int8, device="cuda")
        w = torch.empty(r1 - r0, gs * gpr, dtype=torch.float32, device="cuda")
        ccq.decode(d, levels=lv, weights=w)
        assert np.array_equal(lv.cpu().numpy(), lv_all[r0:r1]), (r0, r1)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), w_all[r0:r1].view(np.uint32)), (r0, r1)


@pytest.mark.parametrize("fam", [2, 0, 1])
def test_device_loader_multi_chunk_rows(oracle, ccq, cuda, fam):
    """Rows spanning several 32-group chunks with a ragged last chunk (gpr=70)
    and a row count that is not a multiple of 16: decode bit-exact and the
    GEMV/GEMM agree with the oracle after the device re-layout."""
    torch = cuda
    s = oracle.random_packed(37, 64 * 70, fam, 64, seed=5 + fam)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    w = torch.empty(37, 64 * 70, dtype=torch.float32, device="cuda")
    ccq.decode(d, weights=w)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), oracle.dequantize(s).view(np.uint32))
    x = oracle.random_matrix(3, 64 * 70, "gaussian", 6)
    assert rel_err(ccq.gemv_batch(d, x), oracle.gemv_batch(s, x)) < REL_TOL


@pytest.mark.parametrize("M", [3, 5, 8])
def test_k_heavy_206_small_batch_on_gemm(oracle, ccq, cuda, M):
    """2.06 on a K-heavy layer (14336 -> 4096) hands M >= 3 to the split-K
    tcgen05 GEMM (model.cu dispatch): whole output against the tensor-pipe
    GEMV and sampled rows against the oracle."""
    torch = cuda
    s = oracle.random_packed(4096, 14336, 2, 64, seed=14336 + M)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = bf16_round(oracle.random_matrix(M, 14336, "gaussian", 200 + M))
    xt = torch.from_numpy(x).to("cuda").to(torch.bfloat16)
    y = ccq.matmul(d, xt)
    ref = ccq.matmul(d, xt, kernel="gemv")
    torch.cuda.synchronize()
    assert rel_err(y.cpu().numpy(), ref.cpu().numpy()) < REL_TOL
    for r0, r1 in ((0, 16), (4080, 4096)):
        want = oracle.gemv_batch(_slice_rows(oracle, s, r0, r1), x, threads=8)
        assert rel_err(y[:, r0:r1].cpu().numpy(), want) < REL_TOL


@pytest.mark.parametrize("fam", [2, 0, 1])
@pytest.mark.parametrize("E,hits,rows,cols", [(8, [0, 1, 3, 4, 7], 48, 1024 + 64), (8, list(range(8)), 64, 4096),
                                              (64, [3, 9, 17, 20, 33, 40, 51, 63], 48, 2048),
                                              (160, list(range(0, 160)), 16, 512)])
@pytest.mark.parametrize("xdt", ["bf16", "f32"])
def test_experts_one_token_per_expert_streaming(oracle, ccq, cuda, fam, E, hits, rows, cols, xdt):
    """MoE decode with one token per routed expert runs the CUDA-core
    streaming GEMV in grouped mode (gemv.cu: CTA b serves hit expert
    b % nhit, x / y rows at the expert's offset); 160 hit experts exceed the
    SM count and take the tensor-pipe path instead."""
    torch = cuda
    counts = [1 if e in hits else 0 for e in range(E)]
    secs, offs, x, want = _expert_case(oracle, fam, E, rows, cols, counts, seed=E + rows + fam)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s_) for s_ in secs])
    if xdt == "bf16":
        xt = torch.from_numpy(bf16_round(x)).cuda().to(torch.bfloat16)
        for e in range(E):
            if counts[e]:
                want[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], bf16_round(x[offs[e]:offs[e + 1]]), threads=8)
    else:
        xt = torch.from_numpy(x).cuda()
    y = ccq.experts_matmul(ex, offs, xt)
    torch.cuda.synchronize()
    assert rel_err(y.cpu().numpy(), want) < REL_TOL
    yb = ccq.experts_matmul(ex, offs, xt, out_dtype=torch.bfloat16)
    assert rel_err(yb.float().cpu().numpy(), want) < 4e-3


@pytest.mark.parametrize("fam", [2, 0, 1])
@pytest.mark.parametrize("counts,rows,cols", [([2, 0, 1, 2, 0, 0, 1, 2], 48, 1024 + 64), ([2] * 8, 64, 4096),
                                              ([0, 2, 0, 0, 1, 0, 2, 0] * 8, 32, 2048)])
@pytest.mark.parametrize("xdt", ["bf16", "f32"])
def test_experts_two_tokens_per_expert(oracle, ccq, cuda, fam, counts, rows, cols, xdt):
    """Up to two tokens per routed expert (mixed 0 / 1 / 2): routed to the
    grouped tensor-pipe GEMV (a grouped M = 2 streaming variant measured 5x
    slower, profiles/r01_moe_grouped_stream_m2_experiment.txt)."""
    torch = cuda
    E = len(counts)
    secs, offs, x, want = _expert_case(oracle, fam, E, rows, cols, counts, seed=E * 7 + rows + fam)
    ex = ccq.Experts.upload([ccq.PackedModel.from_sections(s_) for s_ in secs])
    if xdt == "bf16":
        xt = torch.from_numpy(bf16_round(x)).cuda().to(torch.bfloat16)
        for e in range(E):
            if counts[e]:
                want[offs[e]:offs[e + 1]] = oracle.gemv_batch(secs[e], bf16_round(x[offs[e]:offs[e + 1]]), threads=8)
    else:
        xt = torch.from_numpy(x).cuda()
    y = ccq.experts_matmul(ex, offs, xt)
    torch.cuda.synchronize()
    assert rel_err(y.cpu().numpy(), want) < REL_TOL


def test_config0_full_size_gaussian_quantized(oracle, ccq, cuda):
    """BASELINE configs[0] as specified: a 4096 x 4096 Gaussian weight matrix
    (the reference's random_matrix, mt19937_64 + Box-Muller) quantized to 2.06
    bits (quantize_tensor, g = 64, rounds = 2) on the GPU, then decode and the
    batch-1 GEMV against the CPU oracle.  The quantization itself is pinned
    to the reference's own quantizer (oracle/_ref) on two 32-row slices (the
    quantizer is row-independent), the decode is bit-exact over the whole
    matrix and the M = 1 products (bf16 and f32 activations) are within the
    reference's acceptance tolerance 1e-4 (acceptance_main.cpp:329-371)."""
    torch = cuda
    w = oracle.random_matrix(4096, 4096, "gaussian", 4096 * 31 + 4096).astype(np.float32)
    got = ccq.quantize(w, 2, 64, 2)
    s = oracle.Sections(got.rows, got.cols, got.family, got.group_size,
                        np.asarray(got.code_payload, np.uint8), np.asarray(got.scale_payload, np.uint8),
                        np.asarray(got.super_scales, np.float32), np.asarray(got.cluster_scales, np.float32),
                        np.asarray(got.cluster_zero_points, np.float32))
    if oracle.ref_available():
        for r0 in (0, 2048):
            want = oracle.RefModel.quantize(np.ascontiguousarray(w[r0:r0 + 32]), 2, 64, 2, threads=0).sections()
            part = _slice_rows(oracle, s, r0, r0 + 32)
            assert np.array_equal(part.code_payload, np.asarray(want.code_payload, np.uint8)), r0
            assert np.array_equal(part.scale_payload, np.asarray(want.scale_payload, np.uint8)), r0
            for a, b in ((part.super_scales, want.super_scales), (part.cluster_scales, want.cluster_scales),
                         (part.cluster_zero_points, want.cluster_zero_points)):
                assert np.array_equal(np.asarray(a, np.float32).view(np.uint32),
                                      np.asarray(b, np.float32).view(np.uint32)), r0
    d = ccq.DeviceModel.upload(got)
    assert np.array_equal(ccq.dequantize(d).view(np.uint32), oracle.dequantize(s).view(np.uint32))
    x = oracle.random_matrix(1, 4096, "uniform", 4096 * 31 + 4096)
    for xin in (x, bf16_round(x)):
        want = oracle.gemv_batch(s, xin, threads=8)
        dt = torch.bfloat16 if xin is not x else torch.float32
        y = ccq.matmul(d, torch.from_numpy(xin).to("cuda").to(dt)).cpu().numpy()
        assert rel_err(y, want) < 1e-4


def test_matmul_rejects_bad_output_buffers(oracle, ccq, cuda):
    """out= must be a contiguous f32/bf16 [M, rows] tensor on the activations'
    device; host gemv outputs must be C-contiguous float32 (no silent overrun)."""
    torch = cuda
    s = oracle.random_packed(32, 128, 2, 64, seed=3)
    d = ccq.DeviceModel.upload(ccq.PackedModel.from_sections(s))
    x = torch.randn(2, 128, device="cuda").to(torch.bfloat16)
    for bad in (torch.empty(2, 32, dtype=torch.float16, device="cuda"), torch.empty(2, 16, device="cuda"),
                torch.empty(32, 2, device="cuda").t(), torch.empty(2, 32)):
        with pytest.raises(ccq.ShapeError):
            ccq.matmul(d, x, out=bad)
    with pytest.raises(ccq.ShapeError):
        ccq.matmul(d, x.cpu())
    with pytest.raises(ccq.ShapeError):
        ccq.gemv(d, np.zeros(128, np.float32), np.zeros(32, np.float64))
    with pytest.raises(ccq.ShapeError):
        ccq.gemv_batch(d, np.zeros((2, 128), np.float32), np.zeros((32, 2), np.float32).T)


def test_fp64_widening_variant_subprocess(cuda):
    """The opt-in FP64-pipe widening (CCQ_W64=1: plans built and verified at
    upload, gemv_stream's dot_206_w64) gives the same M = 1 products as the
    default IMAD.WIDE plan path (bit for bit: same fields, same float ops;
    the split-row tail, which the W64 build does not take, is off in both)."""
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import oracle as O, paper_2507_07145_b200 as P\n"
        "s = O.random_packed(300, 4096, 2, 64, seed=5)\n"
        "d = P.DeviceModel.upload(P.PackedModel.from_sections(s))\n"
        "x = torch.from_numpy(O.random_matrix(1, 4096, 'gaussian', 3)).cuda().to(torch.bfloat16)\n"
        "y = P.matmul(d, x).cpu().numpy()\n"
        "np.save(sys.argv[1], y)\n" % ROOT)
    outs = []
    for w64, name in (("1", "a.npy"), ("0", "b.npy")):
        import os
        import tempfile
        path = os.path.join(tempfile.mkdtemp(), name)
        r = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, CCQ_W64=w64, CCQ_GEMV_TAIL="0"),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
