"""The drop-in C++ headers (include/parafac2/*.hpp): compile the restated
reference tests against them on CPU; run them on the GPU."""
import os
import subprocess

import pytest

from tests.helpers import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT,
           "-L", os.path.join(ROOT, "paper_1703_04219_b200", "lib"), "-lp2g",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1703_04219_b200", "lib")]
    subprocess.check_call(cmd)
    return OUT


def test_dropin_headers_compile(p2g):
    assert os.path.exists(build())


@pytest.mark.gpu
def test_dropin_reference_tests_on_gpu(p2g):
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
