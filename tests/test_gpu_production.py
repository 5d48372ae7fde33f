"""GPU parity in the production launch shapes from WELL-CONDITIONED states.

The flat start psi_0 = 1 makes u = F(p) tiny where d > 0, so the float32 residual d/u* is
ill-conditioned there and the protocol's bar max(1e-4, 4 e32) balloons.  Here every
compared state is I.conditioned_state (sqrt(photons) psi_true (1.2 + 0.2 S), S smooth) or a GPU
iterate reached from it (replaced by a fresh conditioned state when the iterate is ill-conditioned),
and each test ASSERTS e32 < 2.5e-5, so the gradient bar really is the north_star's 1e-4.  Fixtures n128m / n256m hold more frames than the persistent frame kernels have
CTAs / clusters, so the multi-frame loops (shared-memory reuse across frames, accumulated trial sums,
L2 prefetch) are exercised.

* teacher-forced iterations (Alg.1, Eq.3, Eq.6/Eq.8, Eq.7): gradient <= 1e-4,
  alpha (DY complex, DY real, FR, PR+) <= 1e-3, every DeltaF_k within the oracle-side bound
  (tests/_common.check_ls_partials), the same accepted trial;
* 20-iteration warm-start trajectories at N = 128 and N = 256: object <= 1e-3, equal shrinks.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402
from tests._common import FIXTURES, c128, check_ls_partials, get_fixture, rel  # noqa: E402

E32_MAX = 2.5e-5


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2106_07575_b200 import _lib
    return _lib


def conditioned(name):
    psi_true, p, scan, d = get_fixture(name)
    psi_c = I.conditioned_state(psi_true, FIXTURES[name][6]).astype(np.complex64)
    return psi_c, p, scan, d


@pytest.mark.parametrize("name,direction", [("n128", 0), ("n256", 0), ("n128m", 0), ("n256m", 0),
                                            ("n128m", 1), ("n128m", 2), ("n128m", 3), ("n256m", 3)])
def test_teacher_forced_conditioned(L, name, direction):
    psi_c, p, scan, d = conditioned(name)
    d64 = d.astype(np.float64)
    p64 = c128(p)
    psi_true = get_fixture(name)[0]
    pt = L.Ptyger(psi_c, p, scan, d, direction=direction)
    for m in range(4):
        psi_m, g_prev, eta_prev, _, mm = pt.get_state()
        assert mm == m
        fresh = False
        g_ref, alpha_ref, _, rs_ref, u_ref = O.grad_at(c128(psi_m), c128(g_prev), c128(eta_prev), m, p64, scan, d64,
                                                       variant=direction)
        if m > 0 and rel(O.gradient_f32(psi_m, p, scan, d), g_ref) >= E32_MAX:
            # the CG iterate wandered into an ill-conditioned state (measured: e32 1.3e-4 at m = 2 on
            # n256m), where the bar would loosen: teacher-force from a FRESH conditioned psi_m instead,
            # keeping the GPU's real g_{m-1}, eta_{m-1} as the direction history
            fresh = True
            psi_m = I.conditioned_state(psi_true, FIXTURES[name][6], seed=5 + m).astype(np.complex64)
            g_ref, alpha_ref, _, rs_ref, u_ref = O.grad_at(c128(psi_m), c128(g_prev), c128(eta_prev), m, p64, scan,
                                                           d64, variant=direction)
        if m > 0:   # teacher forcing: restart from exactly this state (u = G psi_m recomputed)
            pt.set_state(psi_m, g_prev, eta_prev, m)
        tr = pt.iterate(1)[0]
        e32 = rel(O.gradient_f32(psi_m, p, scan, d), g_ref)
        err = rel(pt.get_gradient(), g_ref)
        print(f"{name} dir {direction} m {m}{' (fresh state)' if fresh else ''}: grad err {err:.2e} "
              f"e32 {e32:.2e} shrinks {tr['shrinks']}")
        assert e32 < E32_MAX, (m, e32)
        assert err <= 1e-4, (m, err, e32)
        assert bool(tr["restarted"]) == bool(rs_ref and m > 0)
        if m > 0 and not rs_ref:
            a_gpu = complex(tr["alpha_re"], tr["alpha_im"])
            assert abs(a_gpu - alpha_ref) <= 1e-3 * abs(alpha_ref) + 1e-12, (m, a_gpu, alpha_ref)
        _, _, eta_m, _, _ = pt.get_state()
        v_ref = O.forward_G(c128(eta_m), p64, scan)
        dF = pt.get_ls_partials()
        # PR+ (R#20) has no descent safeguard: eta may point uphill and every trial fail (stall, R#9)
        assert len(dF) == (32 if tr["stalled"] else tr["shrinks"] + 1)
        refs = check_ls_partials(dF, u_ref, v_ref, d64, tr["shrinks"], tr["stalled"])
        if tr["stalled"]:
            assert all(r > 0 for r in refs)      # the oracle rejects every trial as well
    pt.close()


@pytest.mark.parametrize("name", ["n128", "n128m", "n256m"])
def test_warm_start_trajectory_conditioned(L, name):
    """North_star: <= 1e-3 on the object after 20 iterations, from a warm start (SURVEY 8(c).4 item 1:
    free-running trajectories from the flat start are chaotic), in the production frame kernels."""
    psi_c, p, scan, d = conditioned(name)
    ost, otr = O.run_cg(c128(psi_c), c128(p), scan, d.astype(np.float64), 20)
    pt = L.Ptyger(psi_c, p, scan, d)
    gtr = pt.iterate(20)
    err = rel(pt.get_object(), ost.psi)
    print(f"{name}: shrinks {[t['shrinks'] for t in gtr]}, object err {err:.2e}, "
          f"moved {rel(ost.psi, c128(psi_c)):.2e}")
    assert [t["shrinks"] for t in gtr] == [t.shrinks for t in otr]
    assert err <= 1e-3
    F = [t["F"] for t in gtr]
    assert all(F[i + 1] <= F[i] for i in range(len(F) - 1))
    assert rel(np.array(F), np.array([t.F for t in otr])) <= 1e-6
    pt.close()


SCHEDULES = {
    # margin of the adaptive pass-0 trial count: keff = k*_prev + PTYGER_KEFF_ADD
    "keff": [{"PTYGER_KEFF_ADD": "0"}, {"PTYGER_KEFF_ADD": "3"}, {"PTYGER_KEFF_ADD": "12"}],
    # N = 256: share of the frames on the side kernel (k_ls256_side) next to the four-CTA clusters
    "side": [{"PTYGER_C256_SIDE": "0"}, {"PTYGER_C256_SIDE": "110"}, {"PTYGER_C256_SIDE": "300"}],
}


@pytest.mark.parametrize("name,sched", [("n128m", "keff"), ("n256m", "keff"), ("n256m", "side")])
def test_schedule_does_not_change_the_iteration(L, name, sched, monkeypatch):
    """Eq.7 accepts the FIRST trial gamma_0 tau^k that satisfies the Armijo test; how many trials
    one pass over the far fields evaluates (keff = k*_prev + PTYGER_KEFF_ADD, then the extra passes) and which
    kernel transforms which frame (N = 256: the side kernel's share) are scheduling choices that must not
    change the iteration.  From the flat start psi_0 = 1 (k* jumps, extra passes) and in the production
    kernels with more frames than CTAs / clusters: identical shrinks and restarts, F and the object equal to
    float rounding (the trial sums S_k are accumulated in the same per-pixel order whatever the pass holds;
    the frame -> CTA assignment changes only the order of the fp32 partial sums)."""
    psi_true, p, scan, d = get_fixture(name)
    runs = []
    for env in SCHEDULES[sched]:
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
        tr = pt.iterate(8)
        runs.append(([t["shrinks"] for t in tr], [t["restarted"] for t in tr], np.array([t["F"] for t in tr]),
                     [t["ls_passes"] for t in tr], pt.get_object(), pt.kernel_launches()))
        pt.close()
    print(f"{name} {sched}: shrinks {runs[0][0]}, LS passes {[r[3] for r in runs]}, launches {[r[5] for r in runs]}")
    for r in runs[1:]:
        assert r[0] == runs[0][0] and r[1] == runs[0][1]
        assert rel(r[2], runs[0][2]) <= 1e-9
        assert rel(r[4], runs[0][4]) <= 1e-6
    if sched == "keff":
        assert runs[0][3] != runs[2][3]   # the pass schedules really differed
    else:
        assert runs[0][5] < runs[1][5]    # the side kernel really ran (one more launch per iteration)
