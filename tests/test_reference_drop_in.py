"""Drop-in proof (CPU): the reference's OWN unit test, tests/test_domain.cpp
(11 TEST_CASEs, 3474 checks), compiled unchanged against this repo's headers
(include/modeswitch/) and linked against libmodeswitch.so instead of the
reference's proj/core. doctest is absent from the reference (vendor/ not
shipped), so tests/shim/doctest.h provides the macros that file uses.

Needs /root/reference (this container only; skipped on the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
def test_reference_test_domain_passes_against_this_library(tmp_path):
    exe = tmp_path / "test_domain"
    lib = os.path.join(ROOT, "paper_2605_23057_b200", "lib")
    cmd = ["/usr/bin/g++", "-std=c++20", "-O1",
           "-I", os.path.join(ROOT, "tests", "shim"),
           "-I", os.path.join(ROOT, "include"),
           "-I", REF_TESTS,  # test_util.hpp lives beside the test
           os.path.join(REF_TESTS, "test_domain.cpp"),
           "-L", lib, "-lmodeswitch", f"-Wl,-rpath,{lib}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "test cases: 11 | failed: 0" in r.stdout
    assert "failed checks: 0" in r.stdout
