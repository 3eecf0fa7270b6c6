"""Shared fixtures.  ``-m gpu`` tests need a CUDA device (the B200 box);
everything else runs on the CPU.  Golden vectors under ``tests/golden`` were
produced by running the reference package (see golden/make_golden.py)."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built _ts_gpu.so")


def load_golden(name):
    from paper_1212_2287_b200 import load_model
    g = dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")))
    ens = load_model(os.path.join(GOLDEN_DIR, f"{name}.model.txt"))
    return ens, g


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    ens, g = load_golden(request.param)
    return request.param, ens, g


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False
