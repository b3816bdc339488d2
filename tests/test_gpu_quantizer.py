"""GPU exhaustive code search (ccq_cuda_search_codes, csrc/quantize.cu) against
the reference's own search_codes (quantizer.cpp:36-103, compiled from
/root/reference into oracle/_ref by oracle/Makefile): codes must be
bit-identical, including ties (smallest code wins) and short tails."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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
