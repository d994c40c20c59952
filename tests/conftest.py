"""Shared test setup.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box via gpurun).
Everything else runs on CPU (oracle vs golden vectors, host logic, ABI export
checks, gloo multi-process logic).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    """Build the checkers (oracle/Makefile) when missing; the GPU box uses the
    prebuilt .so files that travel with the snapshot."""
    from oracle import oracle
    try:
        oracle.build()
    except Exception as e:  # pragma: no cover - make missing on exotic hosts
        print("oracle build skipped:", e)
    yield


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
