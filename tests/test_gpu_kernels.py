"""Device kernels through the C ABI vs LAPACK/numpy on the same bytes (needs a B200)."""

import numpy as np
import pytest
from scipy.linalg import lapack

from conftest import rel_err, rng, shifted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _arena(torch, n, nslots, seed=0, scale=1.0):
    from paper_1612_00001_b200.device import Arena

    ar = Arena(n, nslots)
    host = rng(seed).standard_normal((nslots, n, n)) * scale
    for s in range(nslots):
        ar.view(s).copy_(torch.from_numpy(host[s]))
    return ar, host


def _x(a):
    """Column-major (X-world) view of a row-major block = its transpose."""
    return a.T


@pytest.mark.parametrize("n", [64, 200, 256, 1000])
def test_gemm_full_and_windows(torch_cuda, n):
    torch = torch_cuda
    ar, host = _arena(torch, n, 4, seed=n)
    X = [_x(h) for h in host]
    # full product, C_out = C_in - A*B
    ar.gemm([(0, 1, 2, 3)], n, n, n, alpha=-1.0, beta=1.0)
    got = _x(ar.view(3).cpu().numpy())
    want = X[2] - X[0] @ X[1]
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    # windowed: ragged M/N/K with offsets, beta = 0 must not read C_in
    ar.view(2).fill_(float("nan"))
    M, N, K = n // 2 + 3, n // 3 + 5, n // 4 + 7
    a0, b0, c0 = (4, 5), (2, 1), (7, 4)
    ar.gemm([(0, 1, 2, 2)], M, N, K, a0=a0, b0=b0, c0=c0, alpha=1.0, beta=0.0)
    got = _x(ar.view(2).cpu().numpy())
    want = X[0][a0[0]:a0[0] + M, a0[1]:a0[1] + K] @ X[1][b0[0]:b0[0] + K, b0[1]:b0[1] + N]
    win = got[c0[0]:c0[0] + M, c0[1]:c0[1] + N]
    assert np.abs(win - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    from paper_1612_00001_b200.errors import DeviceError

    with pytest.raises(DeviceError):  # odd contiguous-dimension offset: rejected, not faulted
        ar.gemm([(0, 1, 2, 2)], M, N, K, a0=(3, 0), alpha=1.0, beta=0.0)
    ar.close()


@pytest.mark.parametrize("n", [40, 100, 256, 333, 1024])
def test_getrf_matches_lapack(torch_cuda, n):
    torch = torch_cuda
    ar, host = _arena(torch, n, 2, seed=7 + n)
    perm = torch.zeros(2 * n, dtype=torch.int32, device="cuda")
    ipiv = torch.zeros(2 * n, dtype=torch.int32, device="cuda")
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    ar.getrf([0, 1], perm, st, ipiv=ipiv)
    assert st.cpu().tolist() == [0, 0]
    for s in range(2):
        lu, piv, info = lapack.dgetrf(_x(host[s]))
        got = _x(ar.view(s).cpu().numpy())
        np.testing.assert_array_equal(ipiv.cpu().numpy()[s * n:(s + 1) * n], piv)
        assert np.abs(got - lu).max() <= 1e-11 * np.abs(lu).max()
        # pi is the composed permutation: (P X)[x] = X[pi[x]]
        p = perm.cpu().numpy()[s * n:(s + 1) * n]
        L = np.tril(got, -1) + np.eye(n)
        U = np.triu(got)
        assert np.abs(_x(host[s])[p] - L @ U).max() <= 1e-11 * n


@pytest.mark.parametrize("n", [8, 33, 64, 96, 128, 250, 512, 2048])
def test_invert_matches_oracle(torch_cuda, n):
    from oracle import bri_oracle as orc

    torch = torch_cuda
    from paper_1612_00001_b200.device import Arena

    a = shifted(n, 100 + n)
    ar = Arena(n, 3)
    ar.view(0).copy_(torch.from_numpy(a))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ar.invert([(0, 1, 2)], st)
    assert int(st.item()) == 0
    got = ar.view(2).cpu().numpy()
    want = orc.invert_dense(a)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    # input untouched
    np.testing.assert_array_equal(ar.view(0).cpu().numpy(), a)
    ar.close()


@pytest.mark.parametrize("n", [16, 64, 96, 128, 512])
def test_schur_node_matches_fold(torch_cuda, n):
    from oracle import bri_oracle as orc

    torch = torch_cuda
    from paper_1612_00001_b200.device import Arena

    blocks = [shifted(n, 300 + n + i) if i == 0 else rng(400 + n + i).standard_normal((n, n))
              for i in range(4)]
    ar = Arena(n, 7)
    for i, blk in enumerate(blocks):
        ar.view(i).copy_(torch.from_numpy(blk))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ar.schur([(0, 1, 2, 3, 4, 5, 6)], st)
    assert int(st.item()) == 0
    got = ar.view(4).cpu().numpy()
    want = orc.fold(*blocks)  # r - l @ inv(p) @ rt
    assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
    ar.close()


@pytest.mark.parametrize("n", [6, 64, 200])
def test_singular_pivot_status(torch_cuda, n):
    torch = torch_cuda
    from paper_1612_00001_b200.device import Arena

    a = rng(9).standard_normal((n, n))
    a[:, 3] = a[:, 1] * 2.0  # rank deficient
    ar = Arena(n, 3)
    ar.view(0).copy_(torch.from_numpy(a))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ar.invert([(0, 1, 2)], st)
    assert int(st.item()) > 0
    ar.view(0).zero_()
    ar.invert([(0, 1, 2)], st)
    assert int(st.item()) == 1
    ar.view(0).copy_(torch.from_numpy(shifted(n, 1)))
    ar.view(0)[2, 2] = float("nan")
    ar.invert([(0, 1, 2)], st)
    assert int(st.item()) == 1  # max|A| is NaN: every pivot fails the test (core.py:200-209)
    ar.close()


def test_batched_matches_single(torch_cuda):
    torch = torch_cuda
    from paper_1612_00001_b200.device import Arena

    n, cnt = 256, 5
    ar = Arena(n, 7 * cnt)
    for s in range(4 * cnt):
        ar.view(s).copy_(torch.from_numpy(shifted(n, s) if s % 4 == 0 else rng(s).standard_normal((n, n))))
    items = [(4 * i, 4 * i + 1, 4 * i + 2, 4 * i + 3, 4 * cnt + 3 * i, 4 * cnt + 3 * i + 1, 4 * cnt + 3 * i + 2)
             for i in range(cnt)]
    st = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    ar.schur(items, st)
    batched = [ar.view(it[4]).cpu().numpy().copy() for it in items]
    # a lone factorization takes the extended-panel LU schedule (batches of <= 2,
    # capi.cu getrf_device), which rounds differently from the batched one
    for i, it in enumerate(items):
        ar.schur([it], st[:1])
        assert rel_err(ar.view(it[4]).cpu().numpy(), batched[i]) <= 1e-12
    ar.close()


def test_small_node_schedules_bitwise(tmp_path):
    """The small-node kernel's two schedules — the column-cyclic one-barrier-per-column sweep (default)
    and panels of columns factored inside one warp (BRI_SMALL_BLOCKED=1) — apply the same
    fma sequence to every element: full inverses at b = 1 ... 96 (k = 2 ... 4, heavily pivoting and
    diagonally dominant inputs) and a singular-pivot report are identical bit for bit."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)

    def run(extra, name):
        path = str(tmp_path / name)
        e = dict(os.environ, PYTHONPATH=root, **extra)
        subprocess.run([sys.executable, os.path.join(here, "_small_schedules.py"), path], env=e, check=True,
                       timeout=300)
        return np.load(path)

    blocked, cyclic = run({"BRI_SMALL_BLOCKED": "1"}, "blocked.npz"), run({"BRI_SMALL_BLOCKED": "0"}, "cyclic.npz")
    assert sorted(blocked.files) == sorted(cyclic.files) and len(blocked.files) == 25
    for key in blocked.files:
        assert blocked[key].shape == cyclic[key].shape and np.array_equal(blocked[key], cyclic[key]), key
    assert blocked["singular"].dtype == np.uint8 and b"Singular" in blocked["singular"].tobytes()
