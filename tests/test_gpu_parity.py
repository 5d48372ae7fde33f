"""GPU parity of the CUDA path (through the C ABI) against the float64 oracle.

Tolerances:
  * FFT / u = G psi: rel L2 <= 2e-6 (fp32 radix-16 x radix-T FFT, fp64-built twiddles)
  * F: rel <= 2e-6 (fp32 per-pixel terms, fp64 sums)
  * teacher-forced gradient: rel L2 <= max(1e-4, 4 e32), e32 = error of a plain float32
    NumPy evaluation of the same formula on the same state (oracle.gradient_f32)
  * LS partials DeltaF_k: |GPU - oracle| <= 1e-5 * sum|terms|; same accepted k unless
    ambiguous
  * warm-start 20-iteration trajectory: object rel L2 <= 1e-3, equal shrink sequences
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402
from tests._common import FIXTURES, c128, check_ls_partials, get_fixture, rel  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2106_07575_b200 import _lib
    return _lib


# ------------------------------------------------------------------ FFT library

@pytest.mark.parametrize("N", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft2_matches_oracle_and_cufft(L, N, inverse):
    batch = 37
    x = I.random_complex((batch, N, N), seed=N)
    xt = torch.from_numpy(x.astype(np.complex64)).cuda()
    y = L.fft2(xt, inverse=inverse).cpu().numpy()
    ref = O.uifft2(x) if inverse else O.ufft2(x)
    assert rel(y, ref) < 2e-6
    cu = (torch.fft.ifft2 if inverse else torch.fft.fft2)(xt, norm="ortho").cpu().numpy()
    assert rel(y, cu) < 2e-6
    back = L.fft2(L.fft2(xt, inverse=inverse), inverse=not inverse).cpu().numpy()
    assert rel(back, x) < 3e-6


# ------------------------------------------------------------------ forward / objective

@pytest.mark.parametrize("name", list(FIXTURES))
def test_forward_and_objective(L, name):
    psi_true, p, scan, d = get_fixture(name)
    psi0 = np.ones_like(psi_true) * (0.8 + 0.3j) + 0.05 * I.random_complex(psi_true.shape, seed=1)
    pt = L.Ptyger(psi0, p, scan, d)
    psi0c = psi0.astype(np.complex64).astype(np.complex128)
    u_ref = O.forward_G(psi0c, p.astype(np.complex64).astype(np.complex128), scan)
    assert rel(pt.get_farfield(), u_ref) < 2e-6
    _, _, _, F, m = pt.get_state()
    Fref = O.objective_F(u_ref, d.astype(np.float64))
    assert m == 0 and abs(F - Fref) <= 2e-6 * abs(Fref)
    pt.close()


# ------------------------------------------------------------------ teacher-forced iterations

FLAT = ["tiny", "n32", "n64", "n128", "n256"]


@pytest.mark.parametrize("name", FLAT)
@pytest.mark.parametrize("direction", [0, 2])
def test_teacher_forced_iterations(L, name, direction):
    psi_true, p, scan, d = get_fixture(name)
    d64 = d.astype(np.float64)
    p64 = c128(p)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d, direction=direction)
    n_checked_ls = 0
    for m in range(6):
        psi_m, g_prev, eta_prev, F_m, mm = pt.get_state()
        assert mm == m
        # teacher forcing: restart the GPU from exactly this state (u = G psi_m recomputed),
        # so each step is compared from a fresh far field rather than the lazily updated one
        pt.set_state(psi_m, g_prev, eta_prev, m)
        psi64 = c128(psi_m)
        g_ref, alpha_ref, eta_ref, rs_ref, u_ref = O.grad_at(psi64, c128(g_prev), c128(eta_prev), m, p64, scan, d64,
                                                            variant=direction)
        tr = pt.iterate(1)[0]
        g_gpu = pt.get_gradient()
        e32 = rel(O.gradient_f32(psi_m, p, scan, d), g_ref)
        tol = max(1e-4, 4 * e32)
        assert rel(g_gpu, g_ref) <= tol, (m, rel(g_gpu, g_ref), e32)
        # alpha (Eq.8) from the oracle's sums on the GPU state
        if m > 0 and not rs_ref:
            assert abs(complex(tr["alpha_re"], tr["alpha_im"]) - alpha_ref) <= 1e-3 * abs(alpha_ref) + 1e-12
        assert tr["iter"] == m
        # LS partials on the GPU's eta_m (fp64 oracle, difference form); the tolerance comes from
        # oracle quantities only (tests/_common.check_ls_partials)
        _, _, eta_m, _, _ = pt.get_state()
        v_ref = O.forward_G(c128(eta_m), p64, scan)
        dF = pt.get_ls_partials()
        assert len(dF) == (tr["shrinks"] + 1 if not tr["stalled"] else 32)
        check_ls_partials(dF, u_ref, v_ref, d64, tr["shrinks"], tr["stalled"])
        n_checked_ls += len(dF)
        assert np.isfinite(tr["F"]) and tr["gamma"] in [0.5 ** k for k in range(32)] + [0.0]
    assert n_checked_ls > 0
    pt.close()


# ------------------------------------------------------------------ trajectories

def test_warm_start_trajectory_tiny(L):
    psi_true, p, scan, d = get_fixture("tiny")
    d64 = d.astype(np.float64)
    st, _ = O.run_cg(np.ones_like(psi_true), c128(p), scan, d64, 100)
    psi_w = c128(st.psi)
    ost, otr = O.run_cg(psi_w, c128(p), scan, d64, 20)
    pt = L.Ptyger(psi_w, p, scan, d)
    gtr = pt.iterate(20)
    assert [t["shrinks"] for t in gtr] == [t.shrinks for t in otr]
    assert rel(pt.get_object(), ost.psi) <= 1e-3
    F = [t["F"] for t in gtr]
    assert all(F[i + 1] <= F[i] for i in range(len(F) - 1))
    pt.close()


@pytest.mark.parametrize("name", ["n128", "n256"])
def test_free_running_far_field_drift(L, name):
    """Design S updates u <- u + gamma v instead of recomputing G psi: after 8 free iterations the
    cached far field must still match G psi_m (oracle, fp64) to 1e-5 and the gradient the fresh
    oracle gradient to the 1e-3 object-level bar."""
    psi_true, p, scan, d = get_fixture(name)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    pt.iterate(8)
    psi_m, _, _, _, _ = pt.get_state()
    u_ref = O.forward_G(c128(psi_m), c128(p), scan)
    assert rel(pt.get_farfield(), u_ref) <= 1e-5
    pt.close()


def test_monotone_and_deterministic(L):
    psi_true, p, scan, d = get_fixture("n64")
    outs = []
    for _ in range(2):
        pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
        tr = pt.iterate(12)
        F = [t["F"] for t in tr]
        assert all(F[i + 1] <= F[i] for i in range(len(F) - 1))
        outs.append((pt.get_object(), [t["F"] for t in tr]))
        pt.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]   # bitwise reproducible


# ------------------------------------------------------------------ degenerate cases

def test_d_zero_gradient_closed_form(L):
    psi_true, p, scan, d = get_fixture("n64")
    x = (0.9 + 0.2j) * np.ones_like(psi_true)
    pt = L.Ptyger(x, p, scan, np.zeros_like(d))
    pt.iterate(1)
    Ill = O.illumination(c128(p), scan, x.shape)
    assert rel(pt.get_gradient(), Ill * c128(x)) < 2e-6
    pt.close()


def test_stationary_at_noiseless_truth(L):
    psi_true, p, scan, _ = get_fixture("n64")
    d = np.abs(O.forward_G(c128(psi_true), c128(p), scan)) ** 2
    pt = L.Ptyger(psi_true, p, scan, d.astype(np.float32))
    tr = pt.iterate(1)[0]
    g = pt.get_gradient()
    assert np.linalg.norm(g) <= 1e-4 * np.linalg.norm(O.illumination(c128(p), scan, psi_true.shape) * psi_true)
    # at the fixed point DeltaF(gamma) is below fp32 resolution, so which tiny step is accepted is
    # rounding noise (the fp64 oracle accepts gamma = 1); the step itself must be negligible
    assert tr["step_norm"] <= 1e-5 * np.linalg.norm(psi_true) and not tr["stalled"]
    pt.close()


def test_stall_then_restart(L):
    """t = -1e30: no trial can satisfy Eq.7 -> gamma = 0, stalled; the next iteration sees
    g == g_prev bitwise, so <eta, g - g_prev> = 0 and DY restarts (R#9)."""
    psi_true, p, scan, d = get_fixture("tiny")
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d, t=-1e30)
    tr = pt.iterate(2)
    assert tr[0]["stalled"] == 1 and tr[0]["gamma"] == 0.0 and tr[0]["shrinks"] == 32
    assert tr[1]["stalled"] == 1 and tr[1]["restarted"] == 1
    assert np.array_equal(pt.get_object(), np.ones_like(psi_true).astype(np.complex64))
    pt.close()


def test_bad_data_is_rejected(L):
    psi_true, p, scan, d = get_fixture("tiny")
    d = d.copy()
    d[13, 2, 3] = -1.0
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(psi_true, p, scan, d)
    assert ei.value.status == 3 and "frame 13" in str(ei.value)
    d[13, 2, 3] = np.nan
    with pytest.raises(L.PtygerError):
        L.Ptyger(psi_true, p, scan, d)
    # d is uploaded in two parts (first quarter, rest): the first bad frame is named in either part
    d[13, 2, 3] = 1.0
    d[2, 0, 0] = np.inf
    d[40, 5, 5] = -2.0
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(psi_true, p, scan, d)
    assert ei.value.status == 3 and "frame 2 " in str(ei.value)


def test_single_frame_and_device_inputs(L):
    """n = 1 (degenerate scan) and device-resident inputs through the same C ABI."""
    psi_true, p, scan, d = get_fixture("n128")
    sc = scan[:1].copy()
    dd = d[:1]
    pt = L.Ptyger(torch.from_numpy(np.ones_like(psi_true).astype(np.complex64)).cuda(),
                  torch.from_numpy(p.astype(np.complex64)).cuda(), sc, torch.from_numpy(dd).cuda())
    tr = pt.iterate(1)
    g_ref, _ = O.gradient(np.ones_like(psi_true), c128(p), sc, dd.astype(np.float64))
    e32 = rel(O.gradient_f32(np.ones_like(psi_true), p, sc, dd), g_ref)
    assert rel(pt.get_gradient(), g_ref) <= max(1e-4, 4 * e32), (rel(pt.get_gradient(), g_ref), e32)
    tr += pt.iterate(1)
    assert tr[0]["iter"] == 0 and tr[1]["iter"] == 1 and np.isfinite(tr[1]["F"])
    pt.close()


# ------------------------------------------------------------------ f2 / f3: estimator and direction variants

@pytest.mark.parametrize("name", ["n32", "n128", "n256"])
@pytest.mark.parametrize("direction", [0, 3])
def test_teacher_forced_ls_estimator_and_pr(L, name, direction):
    """Least-squares (Gaussian) estimator (R#19) with Dai-Yuan, and Polak-Ribiere+ (f3) with
    it: gradient, beta/alpha, LS partials (difference form ls_delta_ls) and the accepted trial
    against the oracle from the same teacher-forced state."""
    psi_true, p, scan, d = get_fixture(name)
    d64 = d.astype(np.float64)
    p64 = c128(p)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d, direction=direction, estimator=L.EST_LS)
    for m in range(5):
        psi_m, g_prev, eta_prev, F_m, mm = pt.get_state()
        pt.set_state(psi_m, g_prev, eta_prev, m)
        g_ref, alpha_ref, eta_ref, rs_ref, u_ref = O.grad_at(c128(psi_m), c128(g_prev), c128(eta_prev), m, p64,
                                                            scan, d64, variant=direction, est=O.EST_LS)
        F_ref = O.objective_F_ls(u_ref, d64)
        assert abs(F_m - F_ref) <= 2e-6 * abs(F_ref) or m > 0
        tr = pt.iterate(1)[0]
        e32 = rel(O.gradient_f32(psi_m, p, scan, d, est=O.EST_LS), g_ref)
        assert rel(pt.get_gradient(), g_ref) <= max(1e-4, 4 * e32), (m, rel(pt.get_gradient(), g_ref), e32)
        if m > 0 and not rs_ref:
            gg = float(np.sum(np.abs(g_ref) ** 2))
            gp = float(np.sum(np.abs(c128(g_prev)) ** 2))
            assert abs(complex(tr["alpha_re"], tr["alpha_im"]) - alpha_ref) <= 1e-3 * abs(alpha_ref) + 1e-4 * gg / gp
        _, _, eta_m, _, _ = pt.get_state()
        v_ref = O.forward_G(c128(eta_m), p64, scan)
        dF = pt.get_ls_partials()
        check_ls_partials(dF, u_ref, v_ref, d64, tr["shrinks"], tr["stalled"], est=O.EST_LS)
        # F cached after the step is the LS objective at psi_{m+1} by definition
        psi_n, _, _, F_n, _ = pt.get_state()
        F_def = O.objective_F_ls(O.forward_G(c128(psi_n), p64, scan), d64)
        assert abs(F_n - F_def) <= 1e-5 * (np.sum(np.abs(u_ref) ** 2) + np.sum(d64))
    pt.close()


@pytest.mark.parametrize("est", [0, 1])
def test_gradient_descent_steps(L, est):
    """Eq.4 gradient descent (direction GD): psi_{m+1} = psi_m - gamma0 grad F(psi_m), one
    fixed step per iteration (no line search), against oracle.gd_iterate from the same psi.
    Starts near the truth: from a flat object the ML gradient is dominated by d/|u| at
    near-zero far-field pixels and a fixed step is meaningless."""
    psi_true, p, scan, d = get_fixture("n64")
    d64 = d.astype(np.float64)
    p64 = c128(p)
    Ill = O.illumination(p64, scan, psi_true.shape)
    gamma0 = 0.25 / float(Ill.max())
    psi0 = 0.9 * psi_true + 0.05 * I.random_complex(psi_true.shape, seed=7)
    pt = L.Ptyger(psi0, p, scan, d, direction=L.DIR_GD, gamma0=gamma0, estimator=est)
    Fs = []
    for m in range(4):
        psi_m, _, _, _, _ = pt.get_state()
        psi_ref = O.gd_iterate(c128(psi_m), p64, scan, d64, gamma0, est=est)
        e32 = rel(O.gradient_f32(psi_m, p, scan, d, est=est), (c128(psi_m) - psi_ref) / gamma0)
        tr = pt.iterate(1)[0]
        assert tr["shrinks"] == 0 and tr["gamma"] == gamma0 and tr["alpha_re"] == 0.0 and tr["alpha_im"] == 0.0
        step = np.linalg.norm(psi_ref - c128(psi_m))
        got = pt.get_object()
        assert np.linalg.norm(got - psi_ref) <= 2e-6 * np.linalg.norm(psi_ref) + max(1e-4, 4 * e32) * step, (m, e32)
        objective = O.objective_F_ls if est else O.objective_F
        u_new = O.forward_G(c128(got), p64, scan)
        F_def = objective(u_new, d64)
        a2 = np.abs(u_new) ** 2
        scale = np.sum(a2) + np.sum(d64 * (1.0 + np.abs(np.log(np.maximum(a2, 1e-30)))))
        assert abs(tr["F"] - F_def) <= 1e-5 * scale
        Fs.append(tr["F"])
    assert Fs[-1] < Fs[0]
    pt.close()


def test_view_batch_equals_independent_views(L):
    """f1 (3-D view batch): the views are independent 2-D problems, so a ViewBatch iteration of
    every view is bit-identical to running each view alone, and each matches the oracle."""
    w = I.Workload("vtiny", H=64, W=64, N=16, k=7, step=8, jitter=1, seed=9, photons=1e2, views=3)
    views = []
    for v in range(w.views):
        psi_true, p, scan = I.view_inputs(w, v)
        d = I.poisson_counts(w.photons * np.abs(O.forward_G(psi_true, p, scan)) ** 2, w.seed + v)
        views.append((np.ones_like(psi_true), p, scan, np.asarray(d, np.float32)))
    vb = L.ViewBatch(views)
    trs = vb.iterate(3)
    for v, (o, p, scan, d) in enumerate(views):
        pt = L.Ptyger(o, p, scan, d)
        tr = pt.iterate(3)
        assert [t["shrinks"] for t in tr] == [t["shrinks"] for t in trs[v]]
        assert np.array_equal(pt.get_object(), vb.views[v].get_object())
        st, otr = O.run_cg(c128(o), c128(p), scan, d.astype(np.float64), 3)
        assert [t.shrinks for t in otr] == [t["shrinks"] for t in tr]
        assert rel(pt.get_object(), st.psi) <= 1e-3
        pt.close()
    # rotated phantoms: the views really differ
    assert rel(vb.views[0].get_object(), vb.views[1].get_object()) > 1e-3
    vb.close()


def test_kernel_timers_cover_every_launch(L):
    """ptyger_kernel_times: one GRAD and one LS pass-0 launch per iteration, positive durations that
    fit inside the iteration time, and reset semantics."""
    psi_true, p, scan, d = get_fixture("n128")
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    pt.iterate(1)
    pt.kernel_times(reset=True)
    trs = pt.iterate(4)
    it_ms = pt.last_iterate_ms()
    # per-stage device ms in every trace entry: positive, and together the iteration
    for t in trs:
        assert t["ms_grad"] > 0 and t["ms_dir"] > 0 and t["ms_ls"] > 0 and t["ms_update"] > 0 and t["ms_comm"] == 0
    tot = sum(t["ms_grad"] + t["ms_dir"] + t["ms_ls"] + t["ms_update"] for t in trs)
    assert 0.5 * it_ms <= tot <= 1.02 * it_ms, (tot, it_ms)
    kt = pt.kernel_times(reset=True)
    assert kt["k_grad"][1] == 4 and kt["k_ls"][1] == 4
    assert 0 < kt["k_grad"][0] and 0 < kt["k_ls"][0]
    assert kt["k_grad"][0] + kt["k_ls"][0] <= it_ms * 1.05
    assert pt.kernel_times(reset=True) == {"k_grad": (0.0, 0), "k_ls": (0.0, 0)}
    pt.close()
