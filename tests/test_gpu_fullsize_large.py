"""Parity at BASELINE.json's large view (8192^2 object, 256^2 detector, 99 856 frames) on one GPU, in
the launch configuration bench.py times (cluster-of-four LS kernel, v-slot GRAD kernel), on outputs
the float64 oracle can compute one by one, plus properties that hold at any size:

* grad F at sampled object pixels after the first iteration, each recomputed from only the frames
  whose window covers it (rel L2 over the sample <= max(1e-4, 4 e32), e32 = the plain float32
  evaluation of the same formula);
* the first iterations decrease F (Eq.7 with t = 0 accepts only non-increasing trials), every gamma
  is a trial of the gamma_0 tau^k sequence, the cached F equals the running sum of the accepted DeltaF.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402


@pytest.fixture(scope="module")
def large_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if torch.cuda.get_device_properties(0).total_memory < 170e9:
        pytest.skip("large view needs ~160 GB of device memory")
    import bench
    from paper_2106_07575_b200 import _lib as L
    w = I.WORKLOADS["large"]
    dev = torch.device("cuda", 0)
    psi_true, p, scan, d = bench.synth_device(w, dev)
    psi0 = torch.ones((w.H, w.W), dtype=torch.complex64, device=dev)
    pt = L.Ptyger(psi0, torch.from_numpy(p.astype(np.complex64)).to(dev), scan, d)
    _, _, _, F0, _ = pt.get_state()
    trs = [pt.iterate(1)[0]]
    g = pt.get_gradient()
    trs += pt.iterate(2)
    pt.close()
    return dict(w=w, p=p.astype(np.complex64).astype(np.complex128), scan=scan, d=d, g=g, F0=F0, trs=trs)


def test_large_gradient_sampled_pixels(large_run):
    r = large_run
    scan, p, N = r["scan"], r["p"], r["w"].N
    rng = np.random.default_rng(2)
    lo, hi = int(scan[:, 0].min()), int(scan[:, 0].max()) + N
    pix = np.stack([rng.integers(lo, hi, 8), rng.integers(lo, hi, 8)], 1)
    pix = np.concatenate([pix, [[lo, lo], [hi - 1, hi - 1]]])
    p32 = p.astype(np.complex64)
    u32 = np.fft.fft2(p32, norm="ortho").astype(np.complex64)     # psi_0 = 1: every window is 1
    a2 = (u32.real ** 2 + u32.imag ** 2).astype(np.float32)
    u64 = O.ufft2(p * O.extract(np.ones((N, N), np.complex128), (0, 0), N))
    refs, r32s, gots = [], [], []
    for (y, x) in pix:
        cov = np.where((scan[:, 0] <= y) & (y < scan[:, 0] + N) & (scan[:, 1] <= x) & (x < scan[:, 1] + N))[0]
        dcov = r["d"][torch.from_numpy(cov).to(r["d"].device)].cpu().numpy()
        acc, acc32 = 0j, 0j
        for k, j in enumerate(cov):
            yj = np.conj(p) * O.uifft2(O.residual(u64, dcov[k].astype(np.float64)))
            acc += yj[y - scan[j, 0], x - scan[j, 1]]
            q = np.where(a2 >= np.float32(1e-32), dcov[k] / np.where(a2 > 0, a2, 1), 0).astype(np.float32)
            y32 = np.conj(p32) * np.fft.ifft2((u32 - q * u32).astype(np.complex64), norm="ortho")
            acc32 += complex(y32[y - scan[j, 0], x - scan[j, 1]])
        refs.append(acc)
        r32s.append(acc32)
        gots.append(complex(r["g"][y, x]))
    refs, r32s, gots = np.array(refs), np.array(r32s), np.array(gots)
    e32 = np.linalg.norm(r32s - refs) / np.linalg.norm(refs)
    err = np.linalg.norm(gots - refs) / np.linalg.norm(refs)
    assert err <= max(1e-4, 4 * e32), (err, e32)


def test_large_line_search_properties(large_run):
    trs, F = large_run["trs"], large_run["F0"]
    for t in trs:
        assert not t["stalled"] and t["shrinks"] >= 0
        assert t["gamma"] == 0.5 ** t["shrinks"]
        assert t["F"] <= F            # Eq.7 with t = 0: accepted trials never increase F
        F = t["F"]
    assert trs[-1]["F"] < large_run["F0"]
