"""Pins for the oracle's operators Q, F, G, G^H (Eq.1).

None of these re-types the oracle's own formula: each compares against a
brute-force definition, a closed form or an identity that a dropped term,
a wrong sign / index or a transposed operand would break.
"""
import numpy as np
import pytest

from oracle import ptycho as O
from paper_2106_07575_b200 import inputs as I


def brute_dft2(x):
    """O(N^4) literal 2-D DFT, unitary, e^{-2 pi i (k1 n1 + k2 n2)/N}."""
    N = x.shape[0]
    out = np.zeros_like(x, dtype=np.complex128)
    for k1 in range(N):
        for k2 in range(N):
            s = 0j
            for n1 in range(N):
                for n2 in range(N):
                    s += x[n1, n2] * np.exp(-2j * np.pi * (k1 * n1 + k2 * n2) / N)
            out[k1, k2] = s / N
    return out


@pytest.mark.parametrize("N", [2, 4, 8, 16])
def test_ufft2_matches_brute_force(N):
    x = I.random_complex((N, N), seed=N)
    assert np.max(np.abs(O.ufft2(x) - brute_dft2(x))) < 1e-12 * max(1.0, np.max(np.abs(x))) * N


def test_ufft2_closed_forms():
    # constant 1 on 4x4 -> DC = N = 4, others 0; delta -> all 1/N
    X = O.ufft2(np.ones((4, 4), complex))
    assert abs(X[0, 0] - 4) < 1e-14 and np.max(np.abs(X.ravel()[1:])) < 1e-14
    d = np.zeros((4, 4), complex)
    d[0, 0] = 1
    assert np.max(np.abs(O.ufft2(d) - 0.25)) < 1e-15
    # a single plane wave e^{+2 pi i (a n1 + b n2)/N} lands in bin (a, b) with value N
    N = 16
    n1, n2 = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    X = O.ufft2(np.exp(2j * np.pi * (3 * n1 + 5 * n2) / N))
    assert abs(X[3, 5] - N) < 1e-12
    X[3, 5] = 0
    assert np.max(np.abs(X)) < 1e-12


def test_parseval_and_roundtrip():
    x = I.random_complex((3, 32, 32), seed=3)
    X = O.ufft2(x)
    assert abs(np.sum(np.abs(X) ** 2) / np.sum(np.abs(x) ** 2) - 1) < 1e-13
    assert np.max(np.abs(O.uifft2(X) - x)) < 1e-13


def test_extract_scatter_examples():
    obj = np.ones((8, 8), complex)
    assert np.array_equal(O.extract(obj, (0, 0), 4), np.ones((4, 4)))
    obj = np.zeros((8, 8), complex)
    obj[2, 3] = 5
    e = O.extract(obj, (2, 2), 2)
    assert e[0, 1] == 5 and np.count_nonzero(e) == 1
    # index-by-index loop
    obj = I.random_complex((16, 16), seed=7)
    e = O.extract(obj, (3, 5), 4)
    for i in range(4):
        for k in range(4):
            assert e[i, k] == obj[3 + i, 5 + k]
    acc = np.zeros((8, 8), complex)
    O.scatter_add(acc, np.ones((4, 4)), (0, 0))
    O.scatter_add(acc, np.ones((4, 4)), (2, 2))
    assert acc[2, 2] == 2 and acc[3, 3] == 2 and acc[0, 0] == 1 and acc[5, 5] == 1 and acc[6, 6] == 0
    with pytest.raises(IndexError):
        O.extract(obj, (13, 0), 4)


def test_round_positions_examples():
    # S:75-77 and the float32 trap 0.49999997
    got = O.round_positions([[2.4, 3.6], [2.5, 3.5], [-0.4, 0.0], [0.49999997, 1.5]])
    assert got.tolist() == [[2, 4], [3, 4], [0, 0], [0, 2]]


@pytest.mark.parametrize("H,N,n", [(16, 8, 5), (64, 16, 9), (128, 32, 7)])
def test_G_adjoint_identity(H, N, n):
    rng = np.random.default_rng(H + N)
    scan = rng.integers(0, H - N + 1, size=(n, 2))
    p = I.random_complex((N, N), seed=1)
    x = I.random_complex((H, H), seed=2)
    y = I.random_complex((n, N, N), seed=3)
    lhs = np.vdot(O.forward_G(x, p, scan), y)
    rhs = np.vdot(x, O.adjoint_GH(y, p, scan, (H, H)))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def test_GHG_is_illumination_diagonal():
    """F unitary => G^H G = diag(I), I = sum_j |p(rho - s_j)|^2.  Pins the FFT scale,
    the conj on the probe and the scatter offsets all at once."""
    w = I.WORKLOADS["tiny"]
    psi, p, scan = I.workload_inputs(w)
    x = I.random_complex(psi.shape, seed=9)
    out = O.adjoint_GH(O.forward_G(x, p, scan), p, scan, x.shape)
    Ill = O.illumination(p, scan, x.shape)
    assert np.max(np.abs(out - Ill * x)) < 1e-12 * np.max(np.abs(Ill * x))


def test_linearity():
    w = I.WORKLOADS["tiny"]
    _, p, scan = I.workload_inputs(w)
    a = I.random_complex((64, 64), seed=1)
    b = I.random_complex((64, 64), seed=2)
    lhs = O.forward_G(0.3 * a + (0.2 - 1j) * b, p, scan)
    rhs = 0.3 * O.forward_G(a, p, scan) + (0.2 - 1j) * O.forward_G(b, p, scan)
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(lhs))


@pytest.fixture
def scipy_workers():
    O.set_fft_workers(4)
    yield
    O.set_fft_workers(1)


@pytest.mark.parametrize("N", [4, 8, 16])
def test_scipy_backend_matches_brute_force(N, scipy_workers):
    """FFT_WORKERS > 1 switches ufft2 / uifft2 to scipy.fft: the same brute-force pins hold."""
    x = I.random_complex((N, N), seed=N + 1)
    assert np.max(np.abs(O.ufft2(x) - brute_dft2(x))) < 1e-12 * max(1.0, np.max(np.abs(x))) * N
    assert np.max(np.abs(O.uifft2(O.ufft2(x)) - x)) < 1e-13


def test_forward_G_batch_equals_per_frame():
    H, N = 48, 16
    psi = I.random_complex((H, H), seed=4)
    p = I.make_probe(N)
    scan = I.make_scan(H, H, N, 4, 10, 1, 2)
    ref = O.forward_G(psi, p, scan)
    assert np.max(np.abs(O.forward_G_batch(psi, p, scan) - ref)) < 1e-13 * np.max(np.abs(ref))
    O.set_fft_workers(3)
    try:
        assert np.max(np.abs(O.forward_G_batch(psi, p, scan) - ref)) < 1e-12 * np.max(np.abs(ref))
    finally:
        O.set_fft_workers(1)
