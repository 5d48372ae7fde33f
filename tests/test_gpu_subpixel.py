"""GPU parity of fractional scan positions (bilinear windows, reading R#22)
through ptyger_init_subpixel, against the float64 oracle.  Same tolerances as
tests/test_gpu_parity.py: u = G psi rel L2 <= 2e-6, teacher-forced gradient <= max(1e-4, 4 e32)
with e32 from the float32 yardstick of the same bilinear formula, LS partials within 1e-5 of the
scale or their screening bound, the same accepted trial unless ambiguous, warm-start trajectory
<= 1e-3 with identical shrink sequences.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402
from tests._common import check_ls_partials  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def c128(a):
    return np.asarray(a, np.complex64).astype(np.complex128)


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2106_07575_b200 import _lib
    return _lib


FIXTURES = {
    # name: (H, N, k, step, jitter, seed, photons, noisy)
    "s16": (64, 16, 6, 8, 1.5, 31, 1.0, False),
    "s32": (96, 32, 9, 7, 1.5, 32, 1e3, True),       # 81 frames: FPB = 8 ragged tail
    "s64": (192, 64, 9, 15, 2.5, 33, 1e3, True),
    "s128": (320, 128, 7, 31, 2.5, 34, 1e3, True),
    "s256": (384, 256, 5, 31, 2.5, 35, 1e3, True),   # two-pass FFT through the v slot
}


def get_fixture(name):
    H, N, k, step, jit, seed, ph, noisy = FIXTURES[name]
    psi_true = I.make_object(I.siemens_star(H, H))
    p = I.make_probe(N)
    scan = I.make_scan_subpixel(H, H, N, k, step, jit, seed)
    assert np.any(scan != np.floor(scan))
    mean = ph * np.abs(O.forward_G(psi_true, c128(p), scan)) ** 2
    d = I.poisson_counts(mean, seed) if noisy else mean
    return psi_true, p, scan, np.asarray(d, np.float32)


@pytest.mark.parametrize("name", list(FIXTURES))
def test_forward_subpixel(L, name):
    psi_true, p, scan, d = get_fixture(name)
    psi0 = (0.8 + 0.1j) * np.ones_like(psi_true) + 0.05 * I.random_complex(psi_true.shape, seed=1)
    psi0 = c128(psi0)
    pt = L.Ptyger(psi0, p, scan, d)
    u_gpu = pt.get_farfield()
    u_ref = O.forward_G(psi0, c128(p), scan)
    assert rel(u_gpu, u_ref) <= 2e-6
    _, _, _, F, _ = pt.get_state()
    F_ref = O.objective_F(u_ref, d.astype(np.float64))
    assert abs(F - F_ref) <= 2e-6 * abs(F_ref)
    pt.close()


@pytest.mark.parametrize("name", ["s16", "s32", "s128", "s256"])
def test_teacher_forced_subpixel(L, name):
    psi_true, p, scan, d = get_fixture(name)
    d64 = d.astype(np.float64)
    p64 = c128(p)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    for m in range(5):
        psi_m, g_prev, eta_prev, F_m, mm = pt.get_state()
        assert mm == m
        pt.set_state(psi_m, g_prev, eta_prev, m)
        g_ref, alpha_ref, eta_ref, rs_ref, u_ref = O.grad_at(c128(psi_m), c128(g_prev), c128(eta_prev), m, p64,
                                                            scan, d64)
        tr = pt.iterate(1)[0]
        g_gpu = pt.get_gradient()
        e32 = rel(O.gradient_f32(psi_m, p, scan, d), g_ref)
        assert rel(g_gpu, g_ref) <= max(1e-4, 4 * e32), (m, rel(g_gpu, g_ref), e32)
        if m > 0 and not rs_ref:
            assert abs(complex(tr["alpha_re"], tr["alpha_im"]) - alpha_ref) <= 1e-3 * abs(alpha_ref) + 1e-12
        _, _, eta_m, _, _ = pt.get_state()
        v_ref = O.forward_G(c128(eta_m), p64, scan)
        dF = pt.get_ls_partials()
        check_ls_partials(dF, u_ref, v_ref, d64, tr["shrinks"], tr["stalled"])
    pt.close()


def test_integral_float_positions_run_the_integer_path(L):
    H, N = 96, 32
    psi_true = I.make_object(I.siemens_star(H, H))
    p = I.make_probe(N)
    sc = I.make_scan(H, H, N, 9, 7, 1, 8)
    d = np.asarray(I.poisson_counts(1e3 * np.abs(O.forward_G(psi_true, c128(p), sc)) ** 2, 8), np.float32)
    a = L.Ptyger(np.ones_like(psi_true), p, sc, d)
    b = L.Ptyger(np.ones_like(psi_true), p, sc.astype(np.float32), d)
    ta, tb = a.iterate(3), b.iterate(3)
    assert [t["shrinks"] for t in ta] == [t["shrinks"] for t in tb]
    assert np.array_equal(a.get_object(), b.get_object())
    a.close()
    b.close()


def test_warm_start_trajectory_subpixel(L):
    psi_true, p, scan, d = get_fixture("s16")
    d64 = d.astype(np.float64)
    st, _ = O.run_cg(np.ones_like(psi_true), c128(p), scan, d64, 100)
    psi_w = c128(st.psi)
    ost, otr = O.run_cg(psi_w, c128(p), scan, d64, 20)
    pt = L.Ptyger(psi_w, p, scan, d)
    gtr = pt.iterate(20)
    assert [t["shrinks"] for t in gtr] == [t.shrinks for t in otr]
    assert rel(pt.get_object(), ost.psi) <= 1e-3
    pt.close()


def test_subpixel_window_bounds_rejected(L):
    H, N = 64, 16
    psi = np.ones((H, H), np.complex64)
    p = I.make_probe(N)
    d = np.zeros((1, N, N), np.float32)
    # floor(row) + N = H is fine with a zero fraction (and H - N - 0.5 reads rows up to H - 1),
    # not with a nonzero one
    L.Ptyger(psi, p, np.array([[H - N, 3.5]], np.float32), d).close()
    L.Ptyger(psi, p, np.array([[H - N - 0.5, 3.0]], np.float32), d).close()
    with pytest.raises(L.PtygerError) as e:
        L.Ptyger(psi, p, np.array([[H - N + 0.5, 3.0]], np.float32), d).close()
    assert "outside the object" in str(e.value)
    with pytest.raises(L.PtygerError):
        L.Ptyger(psi, p, np.array([[-0.25, 3.0]], np.float32), d).close()
