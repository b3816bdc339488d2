"""CPU-side checks of the drop-in boundary (no GPU compute).

* libccq_b200.so loads and exports every symbol include/ccq_cuda.h declares;
* the host-only entry points (geometry, widening, container reader) agree
  with the reference / oracle and raise the reference's error types.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ccq_cuda.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(ccq_\w+)\s*\(", txt, re.M)))


def test_header_symbols_listed(ccq):
    assert header_symbols() == sorted(ccq.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol(ccq):
    lib = ccq.lib()
    for sym in header_symbols():
        assert hasattr(lib, sym), sym
    out = subprocess.run(["nm", "-D", "--defined-only", ccq.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for sym in header_symbols():
        assert sym in exported, sym


def test_library_is_sm100a_only(ccq):
    out = subprocess.run(["cuobjdump", "--list-elf", ccq.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_geometry_matches_oracle(ccq, oracle):
    for fam in (0, 1, 2):
        for gs in (57, 64, 65, 66, 1, 0, 3, 7, 8, 4):
            try:
                want = oracle.group_geometry(fam, gs)
            except oracle.OracleError:
                with pytest.raises(ccq.ConfigError):
                    ccq.group_geometry(fam, gs)
                continue
            assert ccq.group_geometry(fam, gs) == want


def test_clustered_code_value_goldens(ccq):
    # test_coding.cpp:224-232
    assert ccq.clustered_code_value(200, 1.0, 0.0) == 200
    assert ccq.clustered_code_value(255, np.float32(32767.0 / 255.0), 0.0) == 32767
    assert ccq.clustered_code_value(1, 2.5, 0.0) == 3
    with pytest.raises(ccq.DomainError):
        ccq.clustered_code_value(255, 200.0, 0.0)
    with pytest.raises(ccq.DomainError):
        ccq.clustered_code_value(0, 1.0, -1.0)


@pytest.mark.parametrize("name,fam", [("2.75", 0), ("2.5", 1), ("2.06", 2)])
def test_container_reader_matches_reference_writer(ccq, oracle, name, fam):
    m = ccq.load_model(os.path.join(GOLDEN, f"acc512_{name}.ccq"))
    assert (m.rows, m.cols, m.family, m.group_size, m.rounds) == (512, 512, fam, 64, 2)
    if os.path.exists(oracle.REF_SO):
        r = oracle.RefModel.load(os.path.join(GOLDEN, f"acc512_{name}.ccq")).sections()
        assert np.array_equal(r.code_payload, m.code_payload)
        assert np.array_equal(r.scale_payload, m.scale_payload)
        assert np.array_equal(r.super_scales.view(np.uint32), m.super_scales.view(np.uint32))
        assert np.array_equal(r.cluster_scales.view(np.uint32), m.cluster_scales.view(np.uint32))
        assert np.array_equal(r.cluster_zero_points.view(np.uint32),
                              m.cluster_zero_points.view(np.uint32))


def test_container_reader_format_errors(ccq, tmp_path):
    src = open(os.path.join(GOLDEN, "acc512_2.06.ccq"), "rb").read()
    cases = {
        "bad magic": b"XCQF" + src[4:],
        "unsupported version": src[:4] + b"\x02\x00" + src[6:],
        "shorter than the fixed prologue": src[:8],
        "header length exceeds": src[:8] + (10**6).to_bytes(4, "little") + src[12:],
        "extends past end of file": src[: len(src) - 100],
    }
    for msg, blob in cases.items():
        p = tmp_path / "c.ccq"
        p.write_bytes(blob)
        with pytest.raises(ccq.FormatError, match=msg):
            ccq.load_model(str(p))


def test_python_packed_model_payload_bytes(ccq, oracle):
    s = oracle.random_packed(64, 64, 2, 64, 3)
    assert ccq.model_payload_bytes(ccq.PackedModel.from_sections(s)) == oracle.payload_bytes(s)


def test_product_does_not_reference_oracle():
    """The product path never loads or imports the checker."""
    pkg = os.path.join(ROOT, "paper_2507_07145_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "ccq_oracle" not in txt, f
                assert "libccq_ref" not in txt, f


def test_reference_exact_synthetic_generators(oracle):
    """ccq_synthetic_packed / ccq_synthetic_matrix (the bench harness's
    generators, host code in libccq_b200.so) reproduce the reference's
    random_quantized + pack_model and random_matrix byte for byte: against
    the C oracle restatement and, when built, the compiled reference."""
    import numpy as np
    from paper_2507_07145_b200.synthetic import reference_matrix, reference_packed
    odd = {2: 65, 0: 66, 1: 57}
    for fam in (2, 0, 1):
        for rows, cols, gs, seed in ((37, 256, 64, 5), (14, 4096, 64, 4096 * 31 + 14336), (9, odd[fam] * 3, odd[fam], 3)):
            a = reference_packed(rows, cols, fam, gs, seed)
            b = oracle.random_packed(rows, cols, fam, gs, seed=seed)
            assert np.array_equal(a.code_payload, b.code_payload)
            assert np.array_equal(a.scale_payload, b.scale_payload)
            for x, y in ((a.super_scales, b.super_scales), (a.cluster_scales, b.cluster_scales),
                         (a.cluster_zero_points, b.cluster_zero_points)):
                assert np.array_equal(np.asarray(x, np.float32).view(np.uint32), np.asarray(y, np.float32).view(np.uint32))
            if oracle.ref_available() and gs == 64:
                r = oracle.RefModel.random(rows, cols, fam, gs, seed).sections()
                assert np.array_equal(a.code_payload, np.asarray(r.code_payload, np.uint8))
    for dist in ("gaussian", "uniform"):
        for rows, cols, seed in ((1, 4096, 4096 * 31 + 14336 + 1), (3, 7, 5)):
            assert np.array_equal(reference_matrix(rows, cols, dist, seed).view(np.uint32),
                                  oracle.random_matrix(rows, cols, dist, seed).view(np.uint32))
