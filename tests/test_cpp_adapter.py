"""The C++ binding a reference maintainer adds (include/snapforge_gpu.hpp),
built against the reference's own headers by tests/cpp/Makefile, run on the
GPU: run_pipeline_gpu vs the reference's run_pipeline(v1, deterministic)
(pipeline.hpp:206-303) on the reference's own problem generators and on a
problem file written by its save_problem (harness.hpp:698-780)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "adapter_test")


def test_adapter_binary_built():
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference tree absent: the binary is built where it exists")
    assert os.path.exists(BIN), "run `make -C tests/cpp` (part of __graft_entry__.build())"


@pytest.mark.gpu
def test_cpp_adapter_vs_reference_pipeline():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/adapter_test not built")
    out = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "bcc54_2j8.problem.json")],
                         capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
    assert out.stdout.count("PASS") >= 7
