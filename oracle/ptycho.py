"""Float64 CPU oracle for the PtyGer ML-CG iteration (arXiv 2106.07575).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2106_07575_b200`` + ``libptyger.so``) never
imports, calls or links it, and shares no code, table or constant with it.

Citation convention: ``P:a-b`` = /root/reference/PAPER.md lines a-b,
``S:a-b`` = SPEC.md lines a-b (used only for interface/edge-case readings),
``R#k`` = reading k in DESIGN.md "Readings of the paper".

Everything is written in the paper's order and notation (Alg. 1
P:626-677), plain NumPy in float64.  The only library primitive used as a step
is the unitary 2-D DFT (``numpy.fft.fft2(norm="ortho")``), itself pinned by a
brute-force DFT test (tests/test_oracle_operators.py).

Pins (what fixes each function to something other than itself) are listed in
DESIGN.md "Oracle pins"; every public function below has at least one.
The free-running fp32-vs-fp64 trajectory from a flat start is
"parity unpinned" (chaotic); only teacher-forced steps and
warm-start trajectories are compared with the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

EPS = 1e-16          # modulus guard, R#4
DEN_EPS = 1e-30      # Dai-Yuan restart threshold, R#9

# direction variants (R#6)
DIR_DY_COMPLEX = 0   # alpha exactly as printed in Eq.6/Eq.8
DIR_DY_REAL = 1      # Re(alpha)
DIR_FR = 2           # Fletcher-Reeves ||g||^2/||g_prev||^2 (north_star)


# --------------------------------------------------------------------------
# Operators Q, F, G = F Q and G^H = Q^H F^H           (Eq.1)
# --------------------------------------------------------------------------

def is_subpixel(scan) -> bool:
    """A floating-point scan array selects the fractional-position operators (R#22)."""
    return np.issubdtype(np.asarray(scan).dtype, np.floating)


def extract(psi: np.ndarray, pos, N: int) -> np.ndarray:
    """Window of psi at integer top-left corner pos=(row, col), N x N (R#3).

    Q's windowing half ("element-wise multiplication of probe p and
    exit wave psi at all scan positions").  A floating-point pos selects the
    bilinear window of R#22 (``extract_bilinear``).
    """
    if np.issubdtype(np.asarray(pos).dtype, np.floating):
        return extract_bilinear(psi, pos, N)
    r, c = int(pos[0]), int(pos[1])
    H, W = psi.shape
    if not (0 <= r <= H - N and 0 <= c <= W - N):
        raise IndexError(f"window at {pos} out of bounds for {psi.shape} with N={N}")
    return psi[r:r + N, c:c + N].copy()


def scatter_add(acc: np.ndarray, patch: np.ndarray, pos) -> None:
    """acc[r+i, c+k] += patch[i, k]: adjoint of ``extract`` (Q^H windowing)."""
    if np.issubdtype(np.asarray(pos).dtype, np.floating):
        scatter_add_bilinear(acc, patch, pos)
        return
    r, c = int(pos[0]), int(pos[1])
    N = patch.shape[0]
    H, W = acc.shape
    if not (0 <= r <= H - N and 0 <= c <= W - N):
        raise IndexError(f"window at {pos} out of bounds for {acc.shape} with N={N}")
    acc[r:r + N, c:c + N] += patch


# Fractional scan positions.  Alg.1 takes the positions as float32 h_s
# but the paper never says how a non-integer position samples the object; reading
# R#22: the window is the BILINEAR interpolation of psi at (y + i, x + k), i.e. with
# r0 = floor(y), fy = y - r0 (same for x):
#   window[i, k] = sum_{a, b in {0, 1}} wy_a wx_b psi[r0 + i + a, c0 + k + b],
#   wy_0 = 1 - fy, wy_1 = fy, wx_0 = 1 - fx, wx_1 = fx.
# Taps with weight 0 are not read, so an integral position reproduces ``extract`` exactly.

def _bilinear_taps(pos):
    y, x = float(pos[0]), float(pos[1])
    r0, c0 = math.floor(y), math.floor(x)
    fy, fx = y - r0, x - c0
    taps = []
    for a, wy in ((0, 1.0 - fy), (1, fy)):
        for b, wx in ((0, 1.0 - fx), (1, fx)):
            if wy * wx != 0.0:
                taps.append((r0 + a, c0 + b, wy * wx))
    return taps


def extract_bilinear(psi: np.ndarray, pos, N: int) -> np.ndarray:
    H, W = psi.shape
    out = np.zeros((N, N), dtype=np.result_type(psi.dtype, np.float64))
    for r, c, w in _bilinear_taps(pos):
        if not (0 <= r <= H - N and 0 <= c <= W - N):
            raise IndexError(f"bilinear window at {tuple(pos)} out of bounds for {psi.shape} with N={N}")
        out += w * psi[r:r + N, c:c + N]
    return out


def scatter_add_bilinear(acc: np.ndarray, patch: np.ndarray, pos) -> None:
    """Adjoint of ``extract_bilinear``: the same real weights, scattered (Q^H)."""
    N = patch.shape[0]
    H, W = acc.shape
    for r, c, w in _bilinear_taps(pos):
        if not (0 <= r <= H - N and 0 <= c <= W - N):
            raise IndexError(f"bilinear window at {tuple(pos)} out of bounds for {acc.shape} with N={N}")
        acc[r:r + N, c:c + N] += w * patch


# FFT_WORKERS > 1: the same unitary transform from scipy.fft with that many threads (a library
# primitive of the same step; the pins in tests/test_oracle_operators.py cover both backends).  Used
# by large-size parity checks and the multi-core CPU baseline variant; 1 = NumPy.
FFT_WORKERS = 1


def set_fft_workers(n: int) -> None:
    global FFT_WORKERS
    FFT_WORKERS = max(1, int(n))


def ufft2(x: np.ndarray) -> np.ndarray:
    """Unitary 2-D DFT, e^{-2 pi i k.n/N}, DC at [0,0], no shift (R#1, R#2).

    F in Eq.1.  Scale 1/N per 2-D transform so F^H = F^{-1}.
    Applied over the last two axes.
    """
    if FFT_WORKERS > 1:
        import scipy.fft
        return scipy.fft.fft2(x, norm="ortho", workers=FFT_WORKERS)
    return np.fft.fft2(x, norm="ortho")


def uifft2(x: np.ndarray) -> np.ndarray:
    """Unitary inverse 2-D DFT = F^H ("F^H is the inverse Fourier transform")."""
    if FFT_WORKERS > 1:
        import scipy.fft
        return scipy.fft.ifft2(x, norm="ortho", workers=FFT_WORKERS)
    return np.fft.ifft2(x, norm="ortho")


def forward_G_batch(psi: np.ndarray, probe: np.ndarray, scan: np.ndarray) -> np.ndarray:
    """forward_G with the windows of all frames stacked and transformed in one batched call (same
    arithmetic per frame: p * window, then ufft2 over the last two axes).  Integer positions only."""
    N = probe.shape[0]
    win = np.stack([extract(psi, s, N) for s in scan]) if len(scan) else np.zeros((0, N, N), psi.dtype)
    return ufft2(probe * win)


def forward_G(psi: np.ndarray, probe: np.ndarray, scan: np.ndarray) -> np.ndarray:
    """(G psi)_j = F(p * psi[window s_j]) for every frame j (Eq.1).

    Returns an (n, N, N) complex128 array, frames in input order.
    """
    N = probe.shape[0]
    out = np.empty((len(scan), N, N), dtype=np.complex128)
    for j, s in enumerate(scan):
        out[j] = ufft2(probe * extract(psi, s, N))
    return out


def adjoint_GH(y: np.ndarray, probe: np.ndarray, scan: np.ndarray, shape) -> np.ndarray:
    """G^H y = sum_j scatter_{s_j}( conj(p) * F^H y_j ), ascending j."""
    acc = np.zeros(shape, dtype=np.complex128)
    pc = np.conj(probe)
    for j, s in enumerate(scan):
        scatter_add(acc, pc * uifft2(y[j]), s)
    return acc


def illumination(probe: np.ndarray, scan: np.ndarray, shape) -> np.ndarray:
    """I(rho) = sum_j |p(rho - s_j)|^2, the diagonal of G^H G (closed form, used as a pin)."""
    acc = np.zeros(shape, dtype=np.float64)
    a2 = np.abs(probe) ** 2
    N = probe.shape[0]
    for s in scan:
        r, c = int(s[0]), int(s[1])
        acc[r:r + N, c:c + N] += a2
    return acc


# --------------------------------------------------------------------------
# Objective (Eq.2) and gradient (Eq.3)
# --------------------------------------------------------------------------

def objective_F(far: np.ndarray, d: np.ndarray, eps: float = EPS) -> float:
    """F = sum_{frames, pixels} ( |G psi|^2 - 2 d log|G psi| )   (Eq.2).

    j runs over all detector pixels of all frames (R#13).
    log|u| is guarded as log max(|u|, eps) (R#4).
    """
    a = np.abs(far)
    return float(np.sum(a * a - 2.0 * d * np.log(np.maximum(a, eps))))


def residual(far: np.ndarray, d: np.ndarray, eps: float = EPS) -> np.ndarray:
    """Gpsi - d/(Gpsi)^*  (the bracket of Eq.3), written as u - d u/|u|^2.

    Where |u| < eps the quotient term is dropped, r = u (R#4).
    """
    a2 = np.abs(far) ** 2
    ok = np.sqrt(a2) >= eps
    q = np.zeros_like(far)
    q[ok] = d[ok] * far[ok] / a2[ok]
    return far - q


def gradient(psi, probe, scan, d, eps: float = EPS):
    """Wirtinger gradient dF/dpsi* = G^H( G psi - d/(G psi)^* )   (Eq.3, R#5).

    Returns (grad, far) where far = G psi.
    """
    far = forward_G(psi, probe, scan)
    return adjoint_GH(residual(far, d, eps), probe, scan, psi.shape), far


# --------------------------------------------------------------------------
# Solver pieces: Dai-Yuan direction (Eq.6, Eq.8), line search (Eq.7), update (Eq.5)
# --------------------------------------------------------------------------

def inner(a: np.ndarray, b: np.ndarray) -> complex:
    """<a, b> = sum_i a_i^* b_i over the z object pixels."""
    return complex(np.sum(np.conj(a) * b))


def dai_yuan(g, g_prev, eta_prev, variant: int = DIR_DY_COMPLEX):
    """Search direction eta_m (Eq.6; coefficient alpha_m Eq.8).

    m = 0 (g_prev is None): eta_0 = -g.
    Otherwise alpha = ||g||^2 / <eta_prev, g - g_prev>  (complex as printed, R#6),
    eta = -g + alpha eta_prev.  |den| < 1e-30 or non-finite alpha => restart
    eta = -g (R#9).  Returns (eta, alpha, restarted).
    """
    if g_prev is None or eta_prev is None:
        return -g, 0j, False
    gg = float(np.sum(np.abs(g) ** 2))
    if variant == DIR_FR:
        den = complex(float(np.sum(np.abs(g_prev) ** 2)))
    else:
        den = inner(eta_prev, g - g_prev)
    if abs(den) < DEN_EPS:
        return -g, 0j, True
    alpha = gg / den
    if variant == DIR_DY_REAL or variant == DIR_FR:
        alpha = complex(alpha.real, 0.0)
    if not (math.isfinite(alpha.real) and math.isfinite(alpha.imag)):
        return -g, 0j, True
    return -g + alpha * eta_prev, alpha, False


@dataclass
class LSConfig:
    gamma0: float = 1.0     # gamma^(0) = 1   (Alg.1)
    tau: float = 0.5        # tau = 0.5       (Alg.1)
    t: float = 0.0          # t "usually set to 0"
    max_shrinks: int = 32   # bound on trials, R#9


def line_search(eval_f, f0: float, cfg: LSConfig):
    """Backtracking line search of Eq.7, Eq.7 semantics (R#7).

    Trials gamma_k = gamma0 * tau^k, k = 0..max_shrinks-1 (first trial is gamma0
    itself); accept the first with F(psi + gamma eta) <= F(psi) + gamma t.
    None accepted: gamma = 0, F unchanged, stalled (R#9).
    Returns (gamma, k, f_new, stalled, trials) with trials = [(gamma_k, f_k)].
    """
    trials = []
    gamma = cfg.gamma0
    for k in range(cfg.max_shrinks):
        fk = float(eval_f(gamma))
        trials.append((gamma, fk))
        if fk <= f0 + gamma * cfg.t:
            return gamma, k, fk, False, trials
        gamma = gamma * cfg.tau
    return 0.0, cfg.max_shrinks, f0, True, trials


def ls_delta(u, v, d, gamma: float, eps: float = EPS) -> float:
    """Difference form of the LS objective:  F(psi + gamma eta) - F(psi).

    With u = G psi, v = G eta (G linear, Eq.1) and per pixel a = 2 Re(u^* v),
    b = |v|^2, c = |u|^2:  |u + gamma v|^2 = c + gamma a + gamma^2 b, so
      dF = sum( gamma a + gamma^2 b - d log(1 + (gamma a + gamma^2 b)/c) ).
    Pixels where |u| < eps or |u + gamma v| < eps use the clamped definition
    (log max(., eps)) exactly as objective_F does (R#4).  This is the quantity
    the GPU line search evaluates; pinned against
    objective_F(u + gamma v) - objective_F(u) in tests.
    """
    a = 2.0 * np.real(np.conj(u) * v)
    b = np.abs(v) ** 2
    c = np.abs(u) ** 2
    q = gamma * a + gamma * gamma * b
    cn = c + q
    e2 = eps * eps
    ok = (c >= e2) & (cn >= e2)
    out = np.where(ok, q, 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        lg = np.where(ok, np.log1p(np.where(ok, q / np.where(ok, c, 1.0), 0.0)), 0.0)
    out = out - d * lg
    bad = ~ok
    if np.any(bad):
        out_b = (cn[bad] - c[bad]) - d[bad] * (np.log(np.maximum(cn[bad], e2))
                                                 - np.log(np.maximum(c[bad], e2)))
        out = out.copy()
        out[bad] = out_b
    return float(np.sum(out))


# --------------------------------------------------------------------------
# One CG iteration (Fig.3 four stages GRAD -> DIR -> LS -> Update, P:462-471,
# Alg.1) and the driver.
# --------------------------------------------------------------------------

@dataclass
class CGState:
    psi: np.ndarray                 # psi_m (H x W complex128)
    g_prev: np.ndarray | None = None   # grad F(psi_{m-1})
    eta_prev: np.ndarray | None = None  # eta_{m-1}
    F: float | None = None          # cached F(psi_m) (R#11)
    m: int = 0


@dataclass
class Trace:
    iter: int
    F: float            # F(psi_{m+1}) (accepted trial value)
    gamma: float
    shrinks: int
    alpha: complex
    restarted: bool
    stalled: bool
    step_norm: float    # ||psi_{m+1} - psi_m||_2
    grad_norm: float
    trials: list = field(default_factory=list)


# --------------------------------------------------------------------------
# Least-squares (Gaussian) estimator: "all the techniques introduced in this
# paper are also applicable to the LS estimator".  Reading R#19:
#   F_LS(psi) = sum_j (|G psi|_j - sqrt(d_j))^2,   grad = G^H( G psi - sqrt(d) G psi / |G psi| )
# (Wirtinger), the quotient dropped where |G psi| < eps exactly as for Eq.3 (R#4).
# --------------------------------------------------------------------------
EST_ML = 0
EST_LS = 1


def objective_F_ls(far: np.ndarray, d: np.ndarray, eps: float = EPS) -> float:
    return float(np.sum((np.abs(far) - np.sqrt(d)) ** 2))


def residual_ls(far: np.ndarray, d: np.ndarray, eps: float = EPS) -> np.ndarray:
    a = np.abs(far)
    ok = a >= eps
    q = np.zeros_like(far)
    q[ok] = np.sqrt(d[ok]) * far[ok] / a[ok]
    return far - q


def gradient_ls(psi, probe, scan, d, eps: float = EPS):
    far = forward_G(psi, probe, scan)
    return adjoint_GH(residual_ls(far, d, eps), probe, scan, psi.shape), far


def _estimator(est: int):
    if est == EST_LS:
        return objective_F_ls, gradient_ls
    return objective_F, gradient


# Further direction rules of the CG family the paper cites around Eq.6 (P:443:
# Dai-Yuan, Polak / Polyak): Polak-Ribiere-Polyak with the usual PR+ clipping.
DIR_PR = 3


def polak_ribiere(g, g_prev, eta_prev):
    """beta = max(0, Re<g, g - g_prev> / ||g_prev||^2); eta = -g + beta eta_prev."""
    if g_prev is None or eta_prev is None:
        return -g, 0j, False
    den = float(np.sum(np.abs(g_prev) ** 2))
    if den < DEN_EPS:
        return -g, 0j, True
    beta = max(0.0, float(np.real(inner(g, g - g_prev))) / den)
    return -g + beta * eta_prev, complex(beta, 0.0), False


def direction(g, g_prev, eta_prev, variant: int):
    if variant == DIR_PR:
        return polak_ribiere(g, g_prev, eta_prev)
    return dai_yuan(g, g_prev, eta_prev, variant)


def cg_iterate(state: CGState, probe, scan, d, ls: LSConfig = LSConfig(),
               variant: int = DIR_DY_COMPLEX, eps: float = EPS, est: int = EST_ML):
    """One iteration of Alg.1 with Eq.7 LS semantics (R#7).

    GRAD: g = grad F(psi_m) (Eq.3; LS estimator: R#19).
    DIR: eta = Dai-Yuan(g, g_prev, eta_prev) (Eq.6) or a variant (R#6, f3).
    LS: gamma from line_search, F evaluated BY DEFINITION on
                      G(psi + gamma eta) for every trial.
    UPD:     psi_{m+1} = psi_m + gamma eta (Eq.5); F cached (R#11).
    Returns (new_state, trace, g, eta).
    """
    objective, grad_fn = _estimator(est)
    psi = state.psi
    g, far = grad_fn(psi, probe, scan, d, eps)
    f0 = state.F if state.F is not None else objective(far, d, eps)
    eta, alpha, restarted = direction(g, state.g_prev if state.m > 0 else None,
                                      state.eta_prev if state.m > 0 else None, variant)

    def eval_f(gamma):
        return objective(forward_G(psi + gamma * eta, probe, scan), d, eps)

    gamma, k, f_new, stalled, trials = line_search(eval_f, f0, ls)
    psi_new = psi + gamma * eta
    tr = Trace(iter=state.m, F=f_new, gamma=gamma, shrinks=k, alpha=alpha,
               restarted=restarted, stalled=stalled,
               step_norm=float(np.sqrt(np.sum(np.abs(psi_new - psi) ** 2))),
               grad_norm=float(np.sqrt(np.sum(np.abs(g) ** 2))), trials=trials)
    return CGState(psi=psi_new, g_prev=g, eta_prev=eta, F=f_new, m=state.m + 1), tr, g, eta


def run_cg(psi0, probe, scan, d, iters: int, ls: LSConfig = LSConfig(),
           variant: int = DIR_DY_COMPLEX, eps: float = EPS, est: int = EST_ML):
    """Alg.1 end to end on one worker: iters CG iterations from psi0 (R#10)."""
    st = CGState(psi=np.asarray(psi0, dtype=np.complex128).copy())
    traces = []
    for _ in range(iters):
        st, tr, _, _ = cg_iterate(st, probe, scan, d, ls, variant, eps, est)
        traces.append(tr)
    return st, traces


def gd_iterate(psi, probe, scan, d, gamma: float, eps: float = EPS, est: int = EST_ML):
    """Gradient-descent update psi - gamma grad F (Eq.4)."""
    g, _ = _estimator(est)[1](psi, probe, scan, d, eps)
    return psi - gamma * g


def ls_delta_ls(u, v, d, gamma: float, eps: float = EPS) -> float:
    """LS-estimator difference form: sum (|u + g v| - sqrt d)^2 - (|u| - sqrt d)^2
    = sum q (1 - 2 sqrt(d) / (|u + g v| + |u|)),  q = |u + g v|^2 - |u|^2."""
    un = np.abs(u + gamma * v)
    uo = np.abs(u)
    q = un * un - uo * uo
    s = un + uo
    frac = np.where(s > 0, 2.0 * np.sqrt(d) / np.where(s > 0, s, 1.0), 0.0)
    return float(np.sum(q * (1.0 - frac)))


# --------------------------------------------------------------------------
# Teacher-forcing helpers: what one GPU iteration must produce from a given state
# --------------------------------------------------------------------------

def grad_at(psi, g_prev, eta_prev, m, probe, scan, d, variant=DIR_DY_COMPLEX, eps=EPS, est=EST_ML):
    """From state (psi_m, g_{m-1}, eta_{m-1}, m): g_m, alpha_m, eta_m, restarted, u=G psi_m."""
    g, far = _estimator(est)[1](psi, probe, scan, d, eps)
    eta, alpha, restarted = direction(g, g_prev if m > 0 else None,
                                      eta_prev if m > 0 else None, variant)
    return g, alpha, eta, restarted, far


def ls_at(psi, eta, probe, scan, d, gammas, eps=EPS):
    """Definition-based F(psi + gamma eta) - F(psi) for each gamma in gammas."""
    f0 = objective_F(forward_G(psi, probe, scan), d, eps)
    return [objective_F(forward_G(psi + g * eta, probe, scan), d, eps) - f0 for g in gammas]


def round_positions(raw) -> np.ndarray:
    """Float scan positions (Alg.1 input 'float32 h_s') -> integer top-left
    corners, round half-up computed in double: floor(x + 0.5) (R#3)."""
    raw = np.asarray(raw, dtype=np.float32).astype(np.float64)
    return np.floor(raw + 0.5).astype(np.int64)


def gradient_f32(psi, probe, scan, d, eps: float = EPS, est: int = EST_ML):
    """The same Eq.3 formula evaluated in plain complex64/float32 NumPy (no reordering):
    the 'e32' yardstick of the teacher-forced tolerance (DESIGN.md Parity protocol,
    SURVEY 8(c).4 item 2).  est = EST_LS evaluates the R#19 residual u - sqrt(d) u/|u|
    instead.  Returns grad as complex128 for comparison."""
    psi = np.asarray(psi, np.complex64)
    probe = np.asarray(probe, np.complex64)
    d = np.asarray(d, np.float32)
    N = probe.shape[0]
    sub = is_subpixel(scan)
    acc = np.zeros(psi.shape, np.complex64)
    for j, s in enumerate(scan):
        if sub:   # R#22 bilinear window, weights and taps in float32
            taps = [(r, c, np.float32(w)) for r, c, w in _bilinear_taps(np.asarray(s, np.float32))]
            win = np.zeros((N, N), np.complex64)
            for r, c, w in taps:
                win = (win + w * psi[r:r + N, c:c + N]).astype(np.complex64)
        else:
            r, c = int(s[0]), int(s[1])
            win = psi[r:r + N, c:c + N]
        u = np.fft.fft2(probe * win, norm="ortho").astype(np.complex64)
        a2 = (u.real * u.real + u.imag * u.imag).astype(np.float32)
        ok = a2 >= np.float32(eps) * np.float32(eps)
        q = np.where(ok, d[j] / np.where(ok, a2, np.float32(1)), np.float32(0)).astype(np.float32)
        if est == EST_LS:
            q = np.sqrt(q).astype(np.float32)
        res = (u - q * u).astype(np.complex64)
        y = (np.conj(probe) * np.fft.ifft2(res, norm="ortho")).astype(np.complex64)
        if sub:
            for r, c, w in taps:
                acc[r:r + N, c:c + N] += w * y
        else:
            acc[r:r + N, c:c + N] += y
    return acc.astype(np.complex128)
