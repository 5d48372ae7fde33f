"""Integer stripe partition of scan frames across P ranks + partitioned gradient.

TEST INFRASTRUCTURE ONLY (see oracle/ptycho.py header).

What the paper fixes: diffraction patterns are partitioned and distributed to
GPUs by spatial location (Fig.4 "workload distribution"); the
global objective is the sum of per-GPU partial sums "according to the addition
associativity".  The paper duplicates halo patterns and exchanges
sub-image borders; this build reads that as unique frame ownership
plus an exchange of partial *gradients* on the shared band (R#15), which is
exact in real arithmetic.  The integer rules below are DESIGN.md R#18
(SURVEY 8(e)); the C++ partitioner in libptyger must reproduce them bit for bit.
"""
from __future__ import annotations

import numpy as np

from .ptycho import forward_G, residual, scatter_add, uifft2, EPS


def canonical_order(scan: np.ndarray, N: int) -> np.ndarray:
    """Frame indices sorted by (centre row r_j + N/2, column c_j, index j)."""
    scan = np.asarray(scan)
    n = len(scan)
    keys = [(int(scan[j, 0]) + N // 2, int(scan[j, 1]), j) for j in range(n)]
    keys.sort()
    return np.array([k[2] for k in keys], dtype=np.int64)


def stripe_bounds(scan, N: int, P: int):
    """b_1..b_{P-1}: centre row of the frame at sorted position floor(i n / P)."""
    order = canonical_order(scan, N)
    n = len(order)
    centres = [int(scan[j, 0]) + N // 2 for j in order]
    return [centres[(i * n) // P] for i in range(1, P)]


def feasible(scan, N: int, P: int) -> bool:
    """Every stripe's centre-row height >= N, measured from the smallest centre row
    to the largest centre row + 1 (so a band touches only two ranks)."""
    if P == 1:
        return True
    scan = np.asarray(scan)
    n = len(scan)
    if P > n:
        return False
    c = scan[:, 0].astype(np.int64) + N // 2
    edges = [int(c.min())] + stripe_bounds(scan, N, P) + [int(c.max()) + 1]
    return all(edges[i + 1] - edges[i] >= N for i in range(P))


def max_feasible_P(scan, N: int, P_limit: int = 64) -> int:
    best = 1
    for P in range(1, P_limit + 1):
        if feasible(scan, N, P):
            best = P
    return best


def split_subpixel(scan):
    """Fractional positions (R#22): integer corners floor(x) and whether any fraction is nonzero."""
    s = np.asarray(scan, dtype=np.float64)
    base = np.floor(s).astype(np.int64)
    return base, bool(np.any(s != base))


def partition(scan, H: int, N: int, P: int, foot: int | None = None):
    """Return (frame_rank[n], rows[P][6]) with rows = own_lo, own_hi, ext_lo, ext_hi,
    store_lo, store_hi (half-open row ranges).

    frame rank: the i whose [b_i, b_{i+1}) holds the centre row (b_0 = -inf, b_P = +inf;
    ties at b_i go to stripe i).
    ext_i = [min owned r_j, min(max owned r_j + foot, H)), foot = N (N + 1 rows for the
    bilinear windows of fractional positions, R#22: ``partition_subpixel``).
    own: o_0 = 0, o_P = H, o_i = clamp(b_i, ext_i.lo, ext_{i-1}.hi) when ext_{i-1}
    and ext_i overlap or touch, else o_i = ext_i.lo.
    store_i = [min(ext_i.lo, o_i), max(ext_i.hi, o_{i+1})).
    """
    scan = np.asarray(scan)
    n = len(scan)
    foot = N if foot is None else foot
    if not feasible(scan, N, P):
        raise ValueError(f"P={P} infeasible; max feasible P = {max_feasible_P(scan, N)}")
    b = stripe_bounds(scan, N, P)
    rank = np.zeros(n, dtype=np.int32)
    for j in range(n):
        cr = int(scan[j, 0]) + N // 2
        i = 0
        while i < P - 1 and cr >= b[i]:
            i += 1
        rank[j] = i
    ext = []
    for i in range(P):
        rs = [int(scan[j, 0]) for j in range(n) if rank[j] == i]
        ext.append((min(rs), min(max(rs) + foot, H)))
    o = [0] * (P + 1)
    o[P] = H
    for i in range(1, P):
        lo, hi_prev = ext[i][0], ext[i - 1][1]
        if lo <= hi_prev:
            o[i] = min(max(b[i - 1], lo), hi_prev)
        else:
            o[i] = lo
    rows = []
    for i in range(P):
        st_lo = min(ext[i][0], o[i])
        st_hi = max(ext[i][1], o[i + 1])
        rows.append((o[i], o[i + 1], ext[i][0], ext[i][1], st_lo, st_hi))
    return rank, rows


def partition_subpixel(scan_f, H: int, N: int, P: int):
    """Partition of fractional positions: rows by floor(x), footprint N + 1 if any fraction != 0."""
    base, sub = split_subpixel(scan_f)
    return partition(base, H, N, P, N + 1 if sub else N)


def band(rows, i: int):
    """Rows [ext_{i+1}.lo, ext_i.hi) shared by ranks i and i+1 (empty tuple if none)."""
    lo, hi = rows[i + 1][2], rows[i][3]
    return (lo, hi) if lo < hi else None


def local_gradient(psi, probe, scan, d, rank, rows, i, eps=EPS):
    """Rank i's partial gradient on its storage rows from its owned frames only
    (ascending global frame index), before any band exchange."""
    st_lo, st_hi = rows[i][4], rows[i][5]
    W = psi.shape[1]
    N = probe.shape[0]
    acc = np.zeros((st_hi - st_lo, W), dtype=np.complex128)
    idx = [j for j in range(len(scan)) if rank[j] == i]
    if not idx:
        return acc
    sc = np.asarray(scan)[idx]
    far = forward_G(psi, probe, sc)
    r = residual(far, np.asarray(d)[idx], eps)
    pc = np.conj(probe)
    for k, s in enumerate(sc):
        # storage-local position (a floating-point position keeps its fraction: bilinear, R#22)
        loc = np.array([s[0] - st_lo, s[1]], dtype=sc.dtype)
        scatter_add(acc, pc * uifft2(r[k]), loc)
    return acc


def exchanged_gradients(psi, probe, scan, d, P, eps=EPS):
    """All ranks' gradients after the band exchange (pure Python, no transport)."""
    H = psi.shape[0]
    N = probe.shape[0]
    if np.issubdtype(np.asarray(scan).dtype, np.floating):
        rank, rows = partition_subpixel(scan, H, N, P)
    else:
        rank, rows = partition(scan, H, N, P)
    parts = [local_gradient(psi, probe, scan, d, rank, rows, i, eps) for i in range(P)]
    out = [p.copy() for p in parts]
    for i in range(P - 1):
        bd = band(rows, i)
        if bd is None:
            continue
        lo, hi = bd
        a = parts[i][lo - rows[i][4]:hi - rows[i][4]]
        c = parts[i + 1][lo - rows[i + 1][4]:hi - rows[i + 1][4]]
        out[i][lo - rows[i][4]:hi - rows[i][4]] = a + c
        out[i + 1][lo - rows[i + 1][4]:hi - rows[i + 1][4]] = c + a
    return rank, rows, out
