"""Test configuration: registers the `gpu` marker and makes the repo root and
oracle/ importable. Native libraries are built in-tree only when missing
(the GPU box receives the prebuilt .so files with the snapshot)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def _ensure_built():
    from paper_2605_23057_b200 import build
    if not os.path.exists(build.ENGINE_SO):
        build.build_engine()
    if not os.path.exists(build.HOST_SO):
        build.build_host()
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build.build_oracle()


_ensure_built()


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
