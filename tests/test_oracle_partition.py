"""Pins for the oracle's integer stripe partition and the band-exchanged gradient
(P:493-503 workload distribution, P:601-604 associativity; R#15, R#18)."""
import numpy as np
import pytest

from oracle import partition as Pt
from oracle import ptycho as O
from paper_2106_07575_b200 import inputs as I


def brute_checks(scan, H, N, P):
    rank, rows = Pt.partition(scan, H, N, P)
    n = len(scan)
    # every frame owned exactly once, centre rows monotone across ranks
    assert rank.shape == (n,) and set(np.unique(rank)) == set(range(P))
    c = scan[:, 0] + N // 2
    for i in range(P - 1):
        assert c[rank == i].max() < c[rank == i + 1].min()
    # owned pixel rows partition [0, H) and sit inside the storage rows
    assert rows[0][0] == 0 and rows[-1][1] == H
    for i in range(P):
        own_lo, own_hi, ext_lo, ext_hi, st_lo, st_hi = rows[i]
        if i + 1 < P:
            assert own_hi == rows[i + 1][0]
        assert own_lo <= own_hi and st_lo <= own_lo and own_hi <= st_hi
        # ext is exactly the hull of the owned windows
        r = scan[rank == i, 0]
        assert ext_lo == r.min() and ext_hi == r.max() + N
        assert st_lo <= ext_lo and ext_hi <= st_hi
    # a band touches only two ranks: ext regions of ranks >= 2 apart are disjoint
    for i in range(P):
        for k in range(i + 2, P):
            assert rows[i][3] <= rows[k][2]
    # every storage row covered by another rank's frames lies in an exchanged band
    for i in range(P):
        st_lo, st_hi = rows[i][4], rows[i][5]
        for k in range(P):
            if k == i:
                continue
            lo, hi = max(st_lo, rows[k][2]), min(st_hi, rows[k][3])
            if lo < hi:
                assert abs(i - k) == 1
                b = Pt.band(rows, min(i, k))
                assert b is not None and b[0] <= lo and hi <= b[1]
    return rank, rows


def test_tiny_max_P_is_3():
    w = I.WORKLOADS["tiny"]
    _, _, scan = I.workload_inputs(w)
    assert Pt.max_feasible_P(scan, w.N) == 3          # span 48 -> P <= 3
    with pytest.raises(ValueError):
        Pt.partition(scan, w.H, w.N, 4)
    rank, rows = brute_checks(scan, w.H, w.N, 3)
    # b_1 = centre of sorted frame floor(49/3)=16 (raster row 2) = 24, b_2 = 40
    assert Pt.stripe_bounds(scan, w.N, 3) == [24, 40]
    assert np.bincount(rank).tolist() == [14, 14, 21]


def test_mid_fixture_bounds():
    w = I.WORKLOADS["mid"]
    _, _, scan = I.workload_inputs(w)
    assert Pt.max_feasible_P(scan, w.N, 20) == 15     # span 960 -> P <= 15
    for P in (1, 2, 4, 8):
        brute_checks(scan, w.H, w.N, P)


def test_P1_is_trivial():
    w = I.WORKLOADS["tiny"]
    _, _, scan = I.workload_inputs(w)
    rank, rows = Pt.partition(scan, w.H, w.N, 1)
    assert np.all(rank == 0)
    assert rows[0] == (0, 64, 0, 64, 0, 64)


def test_jittered_and_random_scans():
    rng = np.random.default_rng(5)
    for trial in range(20):
        H, N = 256, 16
        n = int(rng.integers(20, 200))
        scan = np.stack([rng.integers(0, H - N + 1, n), rng.integers(0, H - N + 1, n)], 1)
        Pm = Pt.max_feasible_P(scan, N, 16)
        for P in range(1, Pm + 1):
            if Pt.feasible(scan, N, P):      # feasibility is not monotone in P
                brute_checks(scan, H, N, P)


@pytest.mark.parametrize("P", [2, 3])
def test_band_exchange_reproduces_global_gradient(P):
    """After exchanging partial gradients on the shared bands, every rank's storage rows
    equal the single-worker gradient (P:601-604 associativity, fp64 rounding only)."""
    w = I.WORKLOADS["tiny"]
    psi_true, p, scan = I.workload_inputs(w)
    d = np.abs(O.forward_G(psi_true, p, scan)) ** 2 * 1.3
    psi = np.ones_like(psi_true) * (0.9 + 0.1j)
    g, _ = O.gradient(psi, p, scan, d)
    rank, rows, gl = Pt.exchanged_gradients(psi, p, scan, d, P)
    for i in range(P):
        st_lo, st_hi = rows[i][4], rows[i][5]
        assert np.max(np.abs(gl[i] - g[st_lo:st_hi])) < 1e-12 * np.max(np.abs(g))
    # owned rows tile the full gradient
    tiled = np.concatenate([gl[i][rows[i][0] - rows[i][4]:rows[i][1] - rows[i][4]] for i in range(P)])
    assert np.max(np.abs(tiled - g)) < 1e-12 * np.max(np.abs(g))
    # partial objectives over owned frames sum to the global F
    far = O.forward_G(psi, p, scan)
    parts = [O.objective_F(far[rank == i], d[rank == i]) for i in range(P)]
    assert abs(sum(parts) - O.objective_F(far, d)) < 1e-12 * abs(O.objective_F(far, d))
