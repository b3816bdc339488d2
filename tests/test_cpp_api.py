"""The drop-in C++ API (include/ccq/*.hpp) compiled against libccq_b200.so,
exercised by a C++ test written like the reference's test_kernels.cpp."""
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

CXX = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle")]


def build(tmp_path, src, extra_objs):
    exe = tmp_path / "t"
    cmd = CXX + [os.path.join(ROOT, "tests", "cpp", src), "-o", str(exe)] + extra_objs + [
        "-Wl,-rpath," + os.path.join(ROOT, "paper_2507_07145_b200"),
        "-Wl,-rpath," + os.path.join(ROOT, "oracle", "_build")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_headers_compile_and_link(ccq, oracle, tmp_path):
    """CPU check: the headers are self-contained and every declared C++ symbol
    resolves against libccq_b200.so (link only, no GPU call)."""
    exe = build(tmp_path, "test_kernels_gpu.cpp",
                [os.path.join(ROOT, "paper_2507_07145_b200", "libccq_b200.so"), oracle.ORACLE_SO])
    assert exe.exists()


@pytest.mark.gpu
def test_cpp_reference_style_kernel_tests(ccq, oracle, cuda, tmp_path):
    exe = build(tmp_path, "test_kernels_gpu.cpp",
                [os.path.join(ROOT, "paper_2507_07145_b200", "libccq_b200.so"), oracle.ORACLE_SO])
    out = subprocess.run([str(exe), GOLDEN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failures" in out.stdout
