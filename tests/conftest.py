"""Shared test plumbing: the `gpu` marker, golden fixtures, repo root on sys.path."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)
GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built qsb200 library")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2009_01845_b200 import _native

    _native.load_library()
    return torch


def circuit_from_json(text):
    from paper_2009_01845_b200.circuit import circuit_from_dict

    return circuit_from_dict(json.loads(str(text)))


@pytest.fixture(params=["batched", "planned"])
def mode(request, monkeypatch):
    """Run a parity test through both execution paths of a first Circuit.execute on a mid-size
    state: the grid-synchronised batch (default) and planned fused passes (specialised kernels)."""
    from paper_2009_01845_b200 import engine

    monkeypatch.setattr(engine, "FIRST_RUN_BATCH", request.param == "batched")
    return request.param
