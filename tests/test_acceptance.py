"""The reference's own acceptance gate (proj/tests/acceptance_main.cpp),
compiled UNMODIFIED against the drop-in headers (include/ccq/) and linked so
that every symbol libccq_b200.so defines - coding/packing rules, pack_model,
load_model, dequantize, gemv, gemv_batch, bench_model, ... - resolves to the
B200 library, with the reference's producer side (quantizer, container
writer, metrics, synthetic generator) from oracle/_ref/libccq_producer.so.
Built by `make -C oracle acceptance` (oracle/Makefile) where /root/reference
exists; the binary travels to the GPU box in oracle/_ref/.

Criteria (acceptance_main.cpp:470-481): 1-5, 7 and 9 exercise the format
rules and pack/unpack on the host; 6 (quantizer/kernel bit agreement), 8
(fused GEMV within 1e-4 on 4096x4096 2.75, 4096x1024 2.5, 8192x8192 2.06,
8192x1024 2.75 at M in {1, 4}) run our GPU kernels; 10 drives the CLI
(`ccq_gpu_bench bench`, tools/ccq_gpu_bench.cpp) through CCQ_BIN."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

ACC = os.path.join(ROOT, "oracle", "_ref", "ccq_acceptance")
HOST_CRITERIA = {1, 2, 3, 4, 5, 7, 9}

needs_binary = pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/ccq_acceptance not built")


def _run(env_extra=None, timeout=1200):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([ACC], capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    results = {}
    for line in out.stdout.splitlines():
        m = re.match(r"\[(PASS|FAIL)\]\s+(\d+)\s", line)
        if m:
            results[int(m.group(2))] = (m.group(1) == "PASS", line)
    return out, results


@needs_binary
def test_acceptance_host_criteria_on_drop_in_headers():
    """CPU: the format / pack criteria pass with our coding.hpp / packing.hpp /
    pack_model implementations standing in for the reference's."""
    out, res = _run({"CUDA_VISIBLE_DEVICES": ""}, timeout=600)
    for c in sorted(HOST_CRITERIA):
        assert c in res, out.stdout + out.stderr
        assert res[c][0], res[c][1]


@needs_binary
@pytest.mark.gpu
def test_acceptance_all_ten_criteria(ccq, cuda, tmp_path):
    """GPU: all ten criteria, with criteria 6 and 8 on the B200 kernels and
    criterion 10 on the GPU bench CLI."""
    exe = tmp_path / "ccq"
    lib_dir = os.path.join(ROOT, "paper_2507_07145_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tools", "ccq_gpu_bench.cpp"), "-o", str(exe),
                    os.path.join(lib_dir, "libccq_b200.so"), "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{lib_dir}", "-Wl,-rpath,/usr/local/cuda/lib64"],
                   check=True, capture_output=True, text=True)
    out, res = _run({"CCQ_BIN": str(exe)})
    assert len(res) == 10, out.stdout + out.stderr
    failed = [res[c][1] for c in sorted(res) if not res[c][0]]
    assert not failed, "\n".join(failed) + "\n" + out.stdout
    assert "acceptance: 10/10" in out.stdout
