"""Shared fixtures; registers the `gpu` marker (tests that need a B200)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def shifted(m: int, seed: int) -> np.ndarray:
    return rng(seed).standard_normal((m, m)) + m * np.eye(m)


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN)
    meta = json.loads(bytes(data["meta"]).decode())
    return data, meta


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


def rel_err(x, y) -> float:
    return float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300))


def oracle_with_floor(a, k, targets, seed=123):
    """CPU-oracle blocks plus the reference's own 1-ulp sensitivity per block.

    The floor is how far the reference BRI moves when M is perturbed by one
    ulp (M * (1 + eps * N(0,1))): the irreducible
    disagreement between two correct FP64 implementations that round
    differently.  Parity is asserted against max(1e-9, 8 * floor).
    """
    from oracle import bri_oracle as orc

    pert = a * (1.0 + 2.220446049250313e-16 * rng(seed).standard_normal(a.shape))
    base = orc.invert_full(a, k, memo=True, targets=list(targets))
    moved = orc.invert_full(pert, k, memo=True, targets=list(targets))
    floor = {t: rel_err(moved[t], base[t]) for t in targets}
    return base, floor


# the reference's own suite (tests/reference_suite/vendored) runs through its import shim in a
# subprocess (tests/test_reference_suite.py); it is never collected into this session
collect_ignore_glob = ["reference_suite/*"]
