"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no G, no FFT, no objective):
it only draws phantoms, the probe, scan positions and Poisson counts from given
means.  Recipe (SPEC simkit S:474-518):

* phantom: Siemens star, img = 1 where cos(spokes/2 * theta) > 0 and
  rho < 0.45 min(H, W) (centre excluded), else 0.  The paper's siemens-star test
  image has no published formula; this is R#14's recipe.
* object: psi_true = (1 - 0.3 img) exp(i pi/2 img).
* probe: Gaussian, sigma = N/4, chirp 8: p = exp(-rho^2/(2 sigma^2)) exp(i 2 pi chirp rho^2/N^2),
  rho measured from (N/2, N/2), normalised so sum |p|^2 = N^2 (R#14).
* scan: k x k raster of top-left corners with the given step, integer jitter
  uniform in [-jitter, jitter], clamped to [0, H-N] x [0, W-N].
* data: d = Poisson(photons * |G psi_true|^2) or the noiseless mean; the mean is
  computed by the CALLER (oracle in tests, torch.fft in bench.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    H: int
    W: int
    N: int
    k: int          # raster is k x k frames
    step: int
    jitter: int
    seed: int
    photons: float = 1e3
    views: int = 1

    @property
    def n(self) -> int:
        return self.k * self.k


# BASELINE.json configs (SURVEY 8 size table).  "mid" is the multi-rank parity fixture.
WORKLOADS = {
    "tiny": Workload("tiny", 64, 64, 16, 7, 8, 0, 23, photons=1.0),
    "small": Workload("small", 1024, 1024, 128, 64, 14, 2, 1),
    "paper": Workload("paper", 4096, 4096, 128, 158, 25, 2, 2),
    "large": Workload("large", 8192, 8192, 256, 316, 25, 2, 3),
    "view3d": Workload("view3d", 2048, 2048, 128, 64, 30, 2, 4, views=64),
    "mid": Workload("mid", 1024, 1024, 64, 121, 8, 0, 5),
    # N = 256 profiling stand-in for "large" (same frame size, step and density; 1/19 of the frames)
    "l256p": Workload("l256p", 2048, 2048, 256, 72, 25, 2, 3),
}


def siemens_star(H: int, W: int, spokes: int = 64, rotation: float = 0.0) -> np.ndarray:
    yy, xx = np.meshgrid(np.arange(H) - H / 2.0, np.arange(W) - W / 2.0, indexing="ij")
    rho = np.hypot(yy, xx)
    theta = np.arctan2(yy, xx) + rotation
    img = ((np.cos(spokes / 2.0 * theta) > 0) & (rho < 0.45 * min(H, W)) & (rho > 0))
    return img.astype(np.float64)


def make_object(img: np.ndarray) -> np.ndarray:
    if np.any(img < 0) or np.any(img > 1):
        raise ValueError("phantom must lie in [0, 1]")
    return (1.0 - 0.3 * img) * np.exp(1j * (np.pi / 2.0) * img)


def make_probe(N: int, sigma_frac: float = 0.25, chirp: float = 8.0) -> np.ndarray:
    if N % 2:
        raise ValueError("N must be even")
    yy, xx = np.meshgrid(np.arange(N) - N / 2.0, np.arange(N) - N / 2.0, indexing="ij")
    r2 = yy * yy + xx * xx
    s = sigma_frac * N
    p = np.exp(-r2 / (2 * s * s)) * np.exp(1j * chirp * 2 * np.pi * r2 / (N * N))
    return p * np.sqrt(N * N / np.sum(np.abs(p) ** 2))


def make_scan(H: int, W: int, N: int, k: int, step: int, jitter: int, seed: int) -> np.ndarray:
    if step >= N:
        raise ValueError("step >= N: no overlap")
    if (k - 1) * step > min(H, W) - N:
        raise ValueError("raster does not fit")
    rng = np.random.default_rng(seed)
    rr, cc = np.meshgrid(np.arange(k) * step, np.arange(k) * step, indexing="ij")
    pos = np.stack([rr.ravel(), cc.ravel()], axis=1).astype(np.int64)
    if jitter:
        pos = pos + rng.integers(-jitter, jitter + 1, size=pos.shape)
    pos[:, 0] = np.clip(pos[:, 0], 0, H - N)
    pos[:, 1] = np.clip(pos[:, 1], 0, W - N)
    return pos.astype(np.int32)


def poisson_counts(mean: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed + 1_000_003)
    return rng.poisson(mean).astype(np.float32)


def random_complex(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def smooth_field(shape, seed: int, modes: int = 6) -> np.ndarray:
    """Smooth complex random field (a few low-frequency separable cosine modes, 1..3 periods across
    the image), scaled to max |.| = 1.  Used to build well-conditioned object states."""
    rng = np.random.default_rng(seed)
    H, W = shape
    yy, xx = np.meshgrid(np.arange(H) / H, np.arange(W) / W, indexing="ij")
    out = np.zeros(shape, np.complex128)
    for _ in range(modes):
        a, b = rng.integers(1, 4, 2)
        ph = rng.uniform(0.0, 2.0 * np.pi, 2)
        amp = rng.standard_normal() + 1j * rng.standard_normal()
        out += amp * np.cos(2 * np.pi * a * yy + ph[0]) * np.cos(2 * np.pi * b * xx + ph[1])
    return out / np.abs(out).max()


def conditioned_state(psi_true: np.ndarray, photons: float, seed: int = 5) -> np.ndarray:
    """A well-conditioned object state for parity checks at production sizes:
    sqrt(photons) psi_true (1.2 + 0.2 S), S = smooth_field.  Near the data's scale (R#14: the ML
    solution is ~ sqrt(photons) psi_true) but 20 % off in amplitude with a smooth complex
    modulation, so the gradient is far from zero and G psi has no near-zeros where d > 0 (a white
    perturbation or the flat psi_0 = 1 produces speckle zeros that make the float32 residual
    d/u* ill-conditioned)."""
    return np.sqrt(photons) * psi_true * (1.2 + 0.2 * smooth_field(psi_true.shape, seed))


def workload_inputs(w: Workload):
    """(psi_true, probe, scan) for a workload; data are the caller's job."""
    img = siemens_star(w.H, w.W)
    return make_object(img), make_probe(w.N), make_scan(w.H, w.W, w.N, w.k, w.step, w.jitter, w.seed)


def view_inputs(w: Workload, v: int):
    """View v of a 3-D batch workload: the phantom rotated by v pi / views, scan seed seed + v."""
    img = siemens_star(w.H, w.W, rotation=v * np.pi / max(w.views, 1))
    return make_object(img), make_probe(w.N), make_scan(w.H, w.W, w.N, w.k, w.step, w.jitter, w.seed + v)


def make_scan_subpixel(H: int, W: int, N: int, k: int, step: int, jitter: float, seed: int) -> np.ndarray:
    """Fractional positions: k x k raster + uniform real jitter in
    [-jitter, jitter], clamped so the bilinear window (N + 1 footprint) stays inside; float32."""
    if (k - 1) * step > min(H, W) - N - 1:
        raise ValueError("raster does not fit")
    rng = np.random.default_rng(seed)
    rr, cc = np.meshgrid(np.arange(k) * step, np.arange(k) * step, indexing="ij")
    pos = np.stack([rr.ravel(), cc.ravel()], axis=1).astype(np.float64)
    pos = pos + rng.uniform(-jitter, jitter, size=pos.shape)
    pos[:, 0] = np.clip(pos[:, 0], 0.0, H - N - 1)
    pos[:, 1] = np.clip(pos[:, 1], 0.0, W - N - 1)
    return pos.astype(np.float32)
