"""Helpers shared by the GPU parity tests: seeded fixtures (data from the float64 oracle), relative
errors, and the line-search tolerance computed from ORACLE quantities only.

Nothing here reads a value produced by the CUDA path: the tolerance of a GPU DeltaF_k is derived
from the oracle's far fields u = G psi, v = G eta and the data d (DESIGN.md "Line search (screen,
then certify)" bound, evaluated on the oracle side with the largest trial set a pass can hold).
"""
import numpy as np

from oracle import ptycho as O
from paper_2106_07575_b200 import inputs as I

LS_EPS_D = 2e-6     # DESIGN.md screening bound constants (MUFU lg2 + fp32 rounding of the sums)
LS_EPS_R = 2e-6
K_PASS = 16         # trials a pass can hold (KC): the bound below maximises over all of them

FIXTURES = {
    # name: (H, N, k, step, jitter, seed, photons, noisy)
    "tiny": (64, 16, 7, 8, 0, 23, 1.0, False),
    "n32": (96, 32, 9, 8, 1, 3, 1e3, True),        # 81 frames: FPB=8 ragged tail
    "n64": (192, 64, 9, 16, 2, 4, 1e3, True),      # 81 frames: FPB=2 ragged tail, 36 tiles
    "n128": (320, 128, 7, 32, 2, 5, 1e3, True),    # 49 frames, 100 tiles
    "n256": (384, 256, 5, 32, 2, 6, 1e3, True),    # 25 frames
    # frames > grid: the persistent frame loops take several trips (148 CTAs for N = 128; 33
    # clusters of four for the N = 256 LS kernel, 148 CTAs for its GRAD kernel)
    "n128m": (456, 128, 21, 16, 2, 8, 1e3, True),  # 441 frames (3 trips), cov 35
    "n256m": (552, 256, 13, 24, 2, 9, 1e3, True),  # 169 frames (> 148 and > 33 x 4), cov 36
}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def c128(a):
    return np.asarray(a, np.complex64).astype(np.complex128)


def problem(H, N, k, step, jitter=0, seed=0, photons=1.0, noisy=False):
    psi_true = I.make_object(I.siemens_star(H, H))
    p = I.make_probe(N)
    scan = I.make_scan(H, H, N, k, step, jitter, seed)
    mean = photons * np.abs(O.forward_G(psi_true, c128(p), scan)) ** 2
    d = I.poisson_counts(mean, seed) if noisy else mean
    return psi_true, p, scan, np.asarray(d, np.float32)


def get_fixture(name):
    H, N, k, step, jit, seed, ph, noisy = FIXTURES[name]
    return problem(H, N, k, step, jit, seed, ph, noisy)


def ls_scale(u, v, d, gamma):
    """sum |terms| of DeltaF(gamma): the yardstick of the flat 1e-5 bar."""
    return float(np.sum(np.abs(u + gamma * v) ** 2) + np.sum(np.abs(u) ** 2)
                 + 2 * np.sum(np.abs(d * np.log(np.maximum(np.abs(u), 1e-30)))))


def screening_moments(u, v, d, gammas):
    """Oracle-side moments of the screening bound, maximised over the trial set `gammas`:
    A = sum d max_k |ln w_k| (w_k = |u + gamma_k v|^2 / |u|^2), D = sum (d + 0.12 |u|^2),
    sum |a|, sum b (a = 2 Re(u* v), b = |v|^2).  Pixels with |u| = 0 are skipped in A (the GPU sends
    such passes to the exact evaluation)."""
    c = np.abs(u) ** 2
    a = 2.0 * np.real(np.conj(u) * v)
    b = np.abs(v) ** 2
    ok = (c > 0) & (d > 0)
    amax = np.zeros(int(np.count_nonzero(ok)))
    uo, vo, co = u[ok], v[ok], c[ok]
    for g in gammas:
        w = np.abs(uo + g * vo) ** 2 / co
        with np.errstate(divide="ignore"):
            amax = np.maximum(amax, np.abs(np.log(np.maximum(w, 1e-300))))
    return (float(np.sum(d[ok] * amax)), float(np.sum(d + 0.12 * c)), float(np.sum(np.abs(a))), float(np.sum(b)))


def screening_bound(mom, gamma):
    A, D, sa, sb = mom
    return LS_EPS_D * D + LS_EPS_R * (A + gamma * sa + gamma * gamma * sb)


def check_ls_partials(dF, u_ref, v_ref, d64, kstar, stalled, gamma0=1.0, tau=0.5, est=O.EST_ML):
    """Every evaluated DeltaF_k against the fp64 difference form on the GPU's eta:
    |GPU - oracle| <= max(1e-5 sum|terms|, B_k) with B_k the screening bound evaluated from oracle
    quantities over a full pass (no value reported by the CUDA path enters the tolerance); the
    bound itself stays below 1e-4 sum|terms|.  Returns the oracle values and the decision check."""
    gam = [gamma0 * tau ** k for k in range(max(len(dF), K_PASS))]
    mom = screening_moments(u_ref, v_ref, d64, gam[:K_PASS]) if est == O.EST_ML else (0.0, 0.0, 0.0, 0.0)
    refs = []
    for k, val in enumerate(dF):
        g = gam[k]
        ref = O.ls_delta(u_ref, v_ref, d64, g) if est == O.EST_ML else O.ls_delta_ls(u_ref, v_ref, d64, g)
        refs.append(ref)
        scale = ls_scale(u_ref, v_ref, d64, g)
        if est == O.EST_ML:
            B = screening_bound(mom, g)
            assert B <= 1e-4 * scale, (k, B, scale)
        else:
            B = 0.0
        assert abs(val - ref) <= max(1e-5 * scale, B), (k, val, ref, scale, B)
    # decision: the first k with DeltaF_k <= 0 (t = 0), unless a margin is below 1e-5 of the scale
    kref = next((k for k, r in enumerate(refs) if r <= 0), None)
    if kref is not None and not stalled:
        scale = float(np.sum(np.abs(u_ref) ** 2) + np.sum(d64))
        if min(abs(r) for r in refs[:kref + 1]) > 1e-5 * scale:
            assert kstar == kref, (kstar, kref)
    return refs
