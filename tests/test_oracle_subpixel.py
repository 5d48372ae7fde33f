"""Pins for the fractional-position (bilinear window) operators of reading R#22 (
Alg.1 input 'float32 h_s').

Each compares against something other than the oracle's own formula: the integer operators
(integral positions), a closed form (bilinear interpolation reproduces affine functions exactly),
hand-computed half-pixel averages, the adjoint identity, central finite differences of the
objective and the partition rules (C library vs oracle, bit-exact).
"""
import numpy as np
import pytest

from oracle import partition as OP
from oracle import ptycho as O
from paper_2106_07575_b200 import inputs as I


def _fixture(H=64, N=16, k=5, step=8, jitter=0.7, seed=3, photons=50.0):
    psi = O.extract(I.make_object(I.siemens_star(H, H)), (0, 0), H) * 1.0
    p = I.make_probe(N)
    sc = I.make_scan_subpixel(H, H, N, k, step, jitter, seed)
    d = photons * np.abs(O.forward_G(psi, p, sc)) ** 2
    return psi, p, sc, d


def test_integral_float_positions_equal_integer_operators():
    psi, p, _, _ = _fixture()
    sc_i = I.make_scan(64, 64, 16, 5, 8, 2, 4)
    sc_f = sc_i.astype(np.float32)
    assert O.is_subpixel(sc_f) and not O.is_subpixel(sc_i)
    a = O.forward_G(psi, p, sc_i)
    b = O.forward_G(psi, p, sc_f)
    assert np.array_equal(a, b)
    y = I.random_complex(a.shape, seed=9)
    assert np.array_equal(O.adjoint_GH(y, p, sc_i, psi.shape), O.adjoint_GH(y, p, sc_f, psi.shape))


def test_bilinear_window_reproduces_affine_functions():
    # psi(r, c) = al r + be c + ga  =>  window[i, k] = al (y + i) + be (x + k) + ga exactly
    H, N = 40, 8
    al, be, ga = 0.3 - 1.1j, -0.7 + 0.25j, 2.0 + 0.5j
    rr, cc = np.meshgrid(np.arange(H), np.arange(H), indexing="ij")
    psi = al * rr + be * cc + ga
    for y, x in [(3.25, 7.5), (0.0, 0.125), (12.9, 30.999), (20.0, 5.0)]:
        pos = np.array([y, x], dtype=np.float64)
        ii, kk = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        want = al * (y + ii) + be * (x + kk) + ga
        assert np.max(np.abs(O.extract(psi, pos, N) - want)) < 1e-12


def test_half_pixel_shift_is_neighbour_average():
    psi = I.random_complex((20, 20), seed=5)
    w = O.extract(psi, np.array([4.5, 6.0]), 6)
    assert np.max(np.abs(w - 0.5 * (psi[4:10, 6:12] + psi[5:11, 6:12]))) < 1e-15
    w = O.extract(psi, np.array([4.5, 6.5]), 6)
    want = 0.25 * (psi[4:10, 6:12] + psi[5:11, 6:12] + psi[4:10, 7:13] + psi[5:11, 7:13])
    assert np.max(np.abs(w - want)) < 1e-15
    # the last row / column may be the window's edge when the fraction is 0 ...
    O.extract(psi, np.array([14.0, 14.0]), 6)
    # ... but not when the bilinear +1 tap is needed
    with pytest.raises(IndexError):
        O.extract(psi, np.array([14.5, 3.0]), 6)


@pytest.mark.parametrize("N,H,k,step", [(8, 40, 4, 6), (16, 64, 5, 8)])
def test_adjoint_identity_subpixel(N, H, k, step):
    p = I.make_probe(N)
    sc = I.make_scan_subpixel(H, H, N, k, step, 1.3, seed=N)
    x = I.random_complex((H, H), seed=1)
    y = I.random_complex((len(sc), N, N), seed=2)
    lhs = np.vdot(O.forward_G(x, p, sc), y)
    rhs = np.vdot(x, O.adjoint_GH(y, p, sc, x.shape))
    assert abs(lhs - rhs) < 1e-10 * abs(lhs)


def test_subpixel_gradient_matches_finite_differences():
    psi, p, sc, d = _fixture(photons=30.0)
    psi0 = psi * (1 + 0.05 * I.random_complex(psi.shape, seed=11))
    g, _ = O.gradient(psi0, p, sc, d)
    for seed, unit in [(21, 1.0), (22, 1j)]:
        delta = unit * I.random_complex(psi.shape, seed=seed)
        h = 1e-6
        fp = O.objective_F(O.forward_G(psi0 + h * delta, p, sc), d)
        fm = O.objective_F(O.forward_G(psi0 - h * delta, p, sc), d)
        fd = (fp - fm) / (2 * h)
        an = 2.0 * np.real(np.vdot(g, delta))
        assert abs(fd - an) < 1e-6 * abs(an)


def test_subpixel_cg_monotone_and_stationary_at_truth():
    psi, p, sc, d = _fixture(photons=1.0)
    # noiseless data: the truth is a stationary point (zero gradient up to rounding)
    g, _ = O.gradient(psi, p, sc, d)
    assert np.max(np.abs(g)) < 1e-9
    st, trs = O.run_cg(np.ones_like(psi), p, sc, d, 6)
    F = [t.F for t in trs]
    assert all(b <= a for a, b in zip(F, F[1:]))


def test_gradient_f32_yardstick_subpixel():
    psi, p, sc, d = _fixture(photons=30.0)
    psi0 = psi * (1 + 0.05 * I.random_complex(psi.shape, seed=12))
    g64, _ = O.gradient(psi0, p, sc, d)
    g32 = O.gradient_f32(psi0, p, sc, d)
    assert np.linalg.norm(g32 - g64) / np.linalg.norm(g64) < 1e-5


def test_partition_subpixel_band_exchange_equals_global_gradient():
    H, N = 256, 16
    psi = I.random_complex((H, H), seed=3)
    p = I.make_probe(N)
    sc = I.make_scan_subpixel(H, H, N, 20, 12, 1.5, seed=7)
    d = 5.0 * np.abs(O.forward_G(psi * 1.1, p, sc)) ** 2
    g, _ = O.gradient(psi, p, sc, d)
    for P in (2, 3, 4):
        rank, rows, parts = OP.exchanged_gradients(psi, p, sc, d, P)
        for i in range(P):
            o_lo, o_hi, _, _, s_lo, _ = rows[i]
            got = parts[i][o_lo - s_lo:o_hi - s_lo]
            assert np.max(np.abs(got - g[o_lo:o_hi])) < 1e-11 * np.max(np.abs(g))
        # the N + 1 footprint: every owned window's last tap row lies inside its storage stripe
        base = np.floor(sc.astype(np.float64)).astype(np.int64)
        for j in range(len(sc)):
            s_lo, s_hi = rows[rank[j]][4], rows[rank[j]][5]
            assert s_lo <= base[j, 0] and base[j, 0] + N + 1 <= s_hi


def test_partition_subpixel_c_matches_oracle():
    from paper_2106_07575_b200 import _lib as L
    rng = np.random.default_rng(0)
    for trial in range(12):
        H, N = int(rng.choice([128, 256, 512])), int(rng.choice([16, 32]))
        k = int(rng.integers(4, 12))
        step = max(1, (H - N - 1) // k)
        sc = I.make_scan_subpixel(H, H, N, k, step, float(rng.uniform(0, 3)), seed=trial)
        if trial % 3 == 0:
            sc = np.floor(sc).astype(np.float32)       # integral: footprint N
        base, _ = OP.split_subpixel(sc)
        for P in range(1, OP.max_feasible_P(base, N, 8) + 1):
            r_o, rows_o = OP.partition_subpixel(sc, H, N, P)
            r_c, rows_c = L.partition_subpixel(sc, H, N, P)
            assert np.array_equal(r_o, r_c)
            assert np.array_equal(np.asarray(rows_o, np.int64), rows_c)
