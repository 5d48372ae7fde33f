"""Shared inputs of the multi-rank GPU tests (seeded; data from the float64 oracle)."""
import numpy as np

from oracle import ptycho as O
from paper_2106_07575_b200 import inputs as I


def fixture(world: int = 2):
    """world <= 5: 256^2 object, 32^2 probe, 20^2 raster with step 10 and jitter 1 (stripes feasible up
    to P = 5); world > 5: 512^2 object, 40^2 raster with step 12 (centre rows span 468: P <= 14)."""
    H, N = (256, 32) if world <= 5 else (512, 32)
    psi_true = I.make_object(I.siemens_star(H, H))
    p = I.make_probe(N)
    scan = I.make_scan(H, H, N, 20, 10, 1, 11) if world <= 5 else I.make_scan(H, H, N, 40, 12, 1, 11)
    mean = 1e3 * np.abs(O.forward_G(psi_true, np.asarray(p, np.complex64).astype(np.complex128), scan)) ** 2
    d = np.asarray(I.poisson_counts(mean, 11), np.float32)
    return np.ones((H, H), np.complex64), p, scan, d
