"""Regression tests for device bugs found in earlier rounds.

Round 1: lu_panel_tall_kernel (panels taller than 8192 rows) read the pivot X(pr, j) from
global memory while rank 0 of the cluster was already swapping rows j and pr — a lagging CTA
scaled its rows by the wrong reciprocal.  It needs interchanges (so the inputs here are plain
Gaussian matrices, not diagonally dominant ones) and skewed CTAs (so half of the repeats run
next to FP64 GEMMs on a side stream, and one run forces the LU's capped persistent GEMMs with
BRI_CAP_ROWS, the round-1 failure condition).  Reference semantics: dgetrf at core.py:249.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe(args, env_extra=None, timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tall_pivot_check.py"), *args],
                         capture_output=True, text=True, env=env, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def cuda_dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


@pytest.mark.parametrize("caps", [None, "1000000"])
def test_tall_panel_heavy_pivoting_dense(cuda_dev, caps):
    """n = 12288 plain Gaussian dense inverse (tall panels + interchanges in nearly every column),
    4 repeats, two of them next to side-stream GEMMs: bit-identical and a tight residual."""
    res = _probe(["--n", "12288", "--repeats", "4"], {"BRI_CAP_ROWS": caps} if caps else None)
    assert res["identical"], res
    # |A X - I| for a Gaussian 12288^2 matrix (cond ~1e4-1e5): ~1e-10; the race gave O(1e-5 .. 1)
    assert max(res["resid"]) <= 1e-7, res


def test_tall_panel_heavy_pivoting_node(cuda_dev):
    """One Schur node of order 10240 (k=2) on a plain Gaussian matrix: the pivot block D and the
    Schur complement both factor through tall panels with heavy pivoting; capped GEMMs forced."""
    res = _probe(["--n", "10240", "--repeats", "3", "--node"], {"BRI_CAP_ROWS": "1000000"})
    assert res["identical"], res
    assert max(res["resid"]) <= 1e-6, res


def test_tall_kernel_small_heavy_pivoting(cuda_dev):
    """The tall-panel kernel forced onto small panels (BRI_TALL_ROWS=256): a plain Gaussian
    n = 1536 dense inverse — interchanges in nearly every column, 16-CTA clusters with only
    ~100 rows each — repeated with and without concurrent GEMMs: bit-identical, tight residual.
    The same configuration is what the compute-sanitizer runs use (profiles/r02_sanitizer_*)."""
    res = _probe(["--n", "1536", "--repeats", "4"], {"BRI_TALL_ROWS": "256"})
    assert res["identical"], res
    assert max(res["resid"]) <= 1e-10, res
