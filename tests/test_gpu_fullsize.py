"""Parity at BASELINE.json's paper-scale view (4096^2 object, 128^2 detector, 24 964 frames), in the
launch configuration bench.py times, from a WELL-CONDITIONED state (I.conditioned_state; the flat
start makes the float32 yardstick e32 balloon), on outputs the float64
oracle can compute one by one:

* u = G psi on sampled frames (rel L2 <= 2e-6);
* grad F at sampled object pixels, each recomputed by the oracle on the sub-problem of only the
  frames whose window covers it (exact: a pixel's gradient depends on nothing else); e32 of the
  same sample asserted < 2.5e-5, so the bar max(1e-4, 4 e32) is 1e-4;
* the first iteration's line-search partials DeltaF_k at the decision boundary (k*-1, k*) over ALL
  frames (oracle far fields of every frame, chunked): within the flat 1e-5 sum|terms| bar, and the
  GPU's accepted trial is the oracle's first accepted one.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402
from tests._common import ls_scale  # noqa: E402


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_view(name, iters_after=0):
    import bench
    from paper_2106_07575_b200 import _lib as L
    w = I.WORKLOADS[name]
    dev = torch.device("cuda", 0)
    psi_true, p, scan, d = bench.synth_device(w, dev)
    psi_c = I.conditioned_state(psi_true, w.photons).astype(np.complex64)
    pt = L.Ptyger(psi_c, torch.from_numpy(p.astype(np.complex64)).to(dev), scan, d)
    _, _, _, F0, _ = pt.get_state()
    idx = np.random.default_rng(0).choice(len(scan), 8, replace=False)
    u0 = pt.get_farfield()[idx] if name == "paper" else None
    tr = pt.iterate(1)[0]
    g = pt.get_gradient()
    _, _, eta, _, _ = pt.get_state()
    dF = pt.get_ls_partials()
    trs = [tr] + (pt.iterate(iters_after) if iters_after else [])
    pt.close()
    return dict(w=w, p=p.astype(np.complex64).astype(np.complex128), scan=scan, d=d, psi=psi_c, idx=idx, u0=u0,
                tr=tr, trs=trs, F0=F0, g=g, eta=eta, dF=dF)


def sampled_gradient(r, pix):
    """(GPU, fp64 oracle, fp32 yardstick) gradient values at the pixels `pix`, the oracle and the
    yardstick evaluated on the cropped sub-problem of the frames covering each pixel."""
    scan, p, N, psi = r["scan"], r["p"], r["w"].N, r["psi"]
    dev_d = r["d"]
    gots, refs, r32s = [], [], []
    for (y, x) in pix:
        cov = np.where((scan[:, 0] <= y) & (y < scan[:, 0] + N) & (scan[:, 1] <= x) & (x < scan[:, 1] + N))[0]
        if len(cov) == 0:      # a pixel no window covers: the gradient is exactly 0 there
            assert r["g"][y, x] == 0
            continue
        r0, c0 = int(scan[cov, 0].min()), int(scan[cov, 1].min())
        r1, c1 = int(scan[cov, 0].max()) + N, int(scan[cov, 1].max()) + N
        crop = psi[r0:r1, c0:c1]
        loc = (scan[cov] - np.array([r0, c0])).astype(np.int32)
        dcov = dev_d[torch.from_numpy(cov).to(dev_d.device)].cpu().numpy()
        g64, _ = O.gradient(crop.astype(np.complex128), p, loc, dcov.astype(np.float64))
        g32 = O.gradient_f32(crop, p.astype(np.complex64), loc, dcov)
        refs.append(g64[y - r0, x - c0])
        r32s.append(g32[y - r0, x - c0])
        gots.append(complex(r["g"][y, x]))
    return np.array(gots), np.array(refs), np.array(r32s)


def boundary_deltas(r, ks, chunk=1024):
    """DeltaF_k (fp64 difference form, oracle.ls_delta) over ALL frames for k in ks, with sum|terms|
    per k.  Far fields by the oracle's batched transform (scipy.fft threads); the elementwise sums
    of each chunk split over a thread pool (NumPy ufuncs release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    scan, p = r["scan"], r["p"]
    psi = r["psi"].astype(np.complex128)
    eta = r["eta"].astype(np.complex128)
    tot = {k: 0.0 for k in ks}
    scale = {k: 0.0 for k in ks}
    nt = cores()

    def part(args):
        u, v, dd = args
        return {k: (O.ls_delta(u, v, dd, 0.5 ** k), ls_scale(u, v, dd, 0.5 ** k)) for k in ks}

    O.set_fft_workers(nt)
    try:
        with ThreadPoolExecutor(nt) as ex:
            for a in range(0, len(scan), chunk):
                sc = scan[a:a + chunk]
                u = O.forward_G_batch(psi, p, sc)
                v = O.forward_G_batch(eta, p, sc)
                dd = r["d"][a:a + chunk].cpu().numpy().astype(np.float64)
                step = max(1, -(-len(sc) // nt))
                for res in ex.map(part, [(u[i:i + step], v[i:i + step], dd[i:i + step])
                                         for i in range(0, len(sc), step)]):
                    for k in ks:
                        tot[k] += res[k][0]
                        scale[k] += res[k][1]
    finally:
        O.set_fft_workers(1)
    return tot, scale


@pytest.fixture(scope="module")
def paper_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return run_view("paper")


def test_farfield_sampled_frames(paper_run):
    r = paper_run
    ref = O.forward_G(r["psi"].astype(np.complex128), r["p"], r["scan"][r["idx"]])
    assert np.linalg.norm(r["u0"] - ref) <= 2e-6 * np.linalg.norm(ref)


def test_gradient_sampled_pixels(paper_run):
    r = paper_run
    scan, N = r["scan"], r["w"].N
    rng = np.random.default_rng(1)
    lo, hi = int(scan[:, 0].min()), int(scan[:, 0].max()) + N
    pix = np.stack([rng.integers(lo, hi, 40), rng.integers(lo, hi, 40)], 1)
    pix = np.concatenate([pix, [[lo, lo], [hi - 1, hi - 1], [lo + N // 2, hi - 1]]])
    gots, refs, r32s = sampled_gradient(r, pix)
    e32 = np.linalg.norm(r32s - refs) / np.linalg.norm(refs)
    err = np.linalg.norm(gots - refs) / np.linalg.norm(refs)
    print(f"paper: sampled gradient err {err:.2e}, e32 {e32:.2e}")
    assert e32 < 2.5e-5, e32
    assert err <= 1e-4, (err, e32)


def test_first_line_search_all_frames(paper_run):
    r = paper_run
    kstar = r["tr"]["shrinks"]
    assert not r["tr"]["stalled"] and len(r["dF"]) == kstar + 1
    ks = [k for k in (kstar - 1, kstar) if k >= 0]      # the decision boundary
    tot, scale = boundary_deltas(r, ks)
    for k in ks:
        print(f"paper: DeltaF_{k} gpu {r['dF'][k]:.9e} oracle {tot[k]:.9e} (rel to scale "
              f"{abs(r['dF'][k] - tot[k]) / scale[k]:.1e})")
        assert abs(r["dF"][k] - tot[k]) <= 1e-5 * scale[k], (k, r["dF"][k], tot[k], scale[k])
    assert tot[kstar] <= 0               # the GPU's accepted trial satisfies Eq.7 (t = 0) ...
    if kstar > 0:
        assert tot[kstar - 1] > 0        # ... and is the first that does
