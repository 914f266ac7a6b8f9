import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


def _ensure_built():
    # Build both the product libraries and the oracle in-tree if missing.
    lib = os.path.join(ROOT, "paper_1801_01572_b200", "_lib", "libloopkit_b200.so")
    syn = os.path.join(ROOT, "paper_1801_01572_b200", "_lib", "libloopkit_synth.so")
    orc = os.path.join(ROOT, "oracle", "_build", "liblk_oracle.so")
    if not (os.path.exists(lib) and os.path.exists(syn)):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1801_01572_b200")], check=True)
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def has_gpu():
    from paper_1801_01572_b200 import device_count
    return device_count() > 0
