"""The C++ host API (include/lbmgpu.hpp) exercised by a compiled C++ program
(tools/cpp_api_test.cpp) written like the reference's doctest kernel tests."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1711_11468_b200", "bin", "cpp_api_test")


@pytest.mark.gpu
def test_cpp_host_api(small_golden):
    fp = {c["snapshot_key"]: c["fingerprint"] for c in small_golden["cases"]
          if c["kind"] == "blocks"}
    r = subprocess.run([EXE, fp["blocks_12x10x10_full"], fp["blocks_12x10x10_half"]],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr


def test_cpp_host_api_builds():
    assert os.path.exists(EXE), "run `make -C tools` (part of __graft_entry__.build())"
