"""Shared pytest setup.

Markers: ``gpu`` — needs a B200 (run by the driver with ``-m gpu``).  Every
other test runs on a CPU-only box (oracle pins, host logic, C-ABI exports,
gloo multi-rank emulation).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA B200 device (sm_100a)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1703_04219_b200", "lib", "libp2g.so")
    ora = os.path.join(ROOT, "oracle", "_build")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1703_04219_b200")])
    if not os.path.isdir(ora) or not any(f.startswith("p2oracle") for f in os.listdir(ora)):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    from tests.helpers import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def p2g():
    import paper_1703_04219_b200 as m

    m.load_library()
    return m


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx(p2g):
    if not _has_gpu():
        pytest.skip("no CUDA device")
    c = p2g.Context(0)
    yield c
    c.close()
