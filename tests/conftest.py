"""Shared test setup: markers, import paths, golden-fixture loaders."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "tests")
GOLDEN = os.path.join(TESTS, "golden")
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpv.so")


def load_json(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_image(name: str) -> np.ndarray:
    """Rebuild a golden memory image from its sparse snapshot."""
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    img = np.zeros(int(z["nbytes"][0]), dtype=np.uint8)
    img.reshape(-1, 4096)[z["pages"].astype(np.int64)] = z["data"]
    return img


def status_outcome(status: int, value: int, aux: int, va: int):
    """Outcome list (tests/scenarios.py format) of a pv.h status word."""
    kind = status & 0xFF0
    level = status & 0xF
    if kind == 0:
        return ["ok", int(value)]
    if kind in (0x010, 0x020):
        return ["fault", int(value), level, 0]
    if kind == 0x040:
        return ["trap", int(va), level, int(value), (status >> 16) & 0x1FF]
    if kind == 0x060:
        return ["trap", int(aux), level, int(value), (status >> 16) & 0x1FF]
    if kind in (0x080, 0x0A0):
        return ["struct"]
    if kind == 0x100:
        return ["oor"]
    return ["unknown", status]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
