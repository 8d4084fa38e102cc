"""Shared fixtures: golden vectors (made by the reference) and markers.

`-m "not gpu"` runs the oracle-vs-golden checks, host logic and C-ABI
symbol checks on CPU; `-m gpu` runs the CUDA parity tests on a B200.
Nothing here reads /root/reference: the golden file was produced there by
tests/golden/make_golden.py and committed.
"""

from __future__ import annotations

import ast
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_PATH = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical runs")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_PATH, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def run_config(golden, i: int) -> dict:
    """GAConfig kwargs of golden whole-loop record i."""
    return dict(ast.literal_eval(str(golden[f"run{i}_cfg"])))


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
