"""`ccq bench`-style CSV for the GPU path (tools/ccq_gpu_bench.cpp, built on the
drop-in C++ API): the reference CLI test checks the CSV schema and the byte
accounting (test_cli.cpp:197-211, kernels.hpp:57-76); the same checks here."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tools", "ccq_gpu_bench.cpp")


def _build(tmp_path):
    exe = tmp_path / "ccq_gpu_bench"
    lib_dir = os.path.join(ROOT, "paper_2507_07145_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           SRC, "-o", str(exe), os.path.join(lib_dir, "libccq_b200.so"), "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{lib_dir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_gpu_bench_cli_builds(ccq, tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_gpu_bench_cli_csv_schema(ccq, oracle, cuda, tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe), "--shapes", "1024x512,4096x4096", "--m", "1,4,40", "--bpw", "2.06",
                          "--iters", "3"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[0] == "shape,M,variant,median_ms,bytes_read"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 2 * 3 * 2
    for shape, m, variant, ms, nbytes in rows:
        d_in, d_out = (int(v) for v in shape.split("x"))
        # model_payload_bytes (kernels.cpp:203-207): codes + nibbles + super + (alpha, beta)
        groups = d_out * d_in // 64
        assert int(nbytes) == groups * 16 + (groups + 1) // 2 + 4 * d_out + 8 * d_out
        assert variant in ("ccq_gpu_fused", "ccq_gpu_fused_e2e")
        assert float(ms) > 0
    bad = subprocess.run([str(exe), "--iters", "0"], capture_output=True, text=True, timeout=60)
    assert bad.returncode == 2  # ConfigError exit code of the reference CLI (ccq_main.cpp:359-366)
