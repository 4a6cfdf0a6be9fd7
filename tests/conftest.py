"""Shared pytest configuration.

Markers: ``gpu`` -- needs a B200 (the parity tests proper, run through the
C ABI).  Everything unmarked runs on the CPU build container.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA B200 device (sm_100a)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1912_02165_b200", "libwinofuse_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", ROOT], check=True)
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def golden_cases():
    with open(os.path.join(GOLDEN, "cases.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN, "cases.npz"))
    out = []
    for m in meta:
        n = m["name"]
        case = dict(m)
        for key in ("x", "w", "pack", "direct", "three_stage", "fused"):
            case[key] = arrays[f"{n}/{key}"]
        out.append(case)
    return out


@pytest.fixture(scope="session")
def golden_basis():
    with open(os.path.join(GOLDEN, "basis.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def cuda_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)
