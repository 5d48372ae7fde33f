"""Parity at BASELINE.json's paper-scale view (4096^2 object, 128^2 detector, 24 964 frames), in
the launch configuration bench.py times, on outputs the float64 oracle can compute one by one:

* u = G psi_0 on sampled frames (rel L2 <= 2e-6);
* grad F at sampled object pixels, each recomputed from only the frames whose window covers it
  (|error| <= 1e-4 of the RMS of the sampled gradient values);
* the first iteration's line-search partials DeltaF_k over ALL frames (oracle evaluated frame
  chunk by frame chunk on the GPU's eta): within max(1e-5 sum|terms|, 2 x the screening bound),
  and the same accepted trial.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ptycho as O  # noqa: E402
from paper_2106_07575_b200 import inputs as I  # noqa: E402


@pytest.fixture(scope="module")
def paper_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import bench
    from paper_2106_07575_b200 import _lib as L
    w = I.WORKLOADS["paper"]
    dev = torch.device("cuda", 0)
    psi_true, p, scan, d = bench.synth_device(w, dev)
    psi0 = torch.ones((w.H, w.W), dtype=torch.complex64, device=dev)
    pt = L.Ptyger(psi0, torch.from_numpy(p.astype(np.complex64)).to(dev), scan, d)
    u0 = pt.get_farfield()
    tr = pt.iterate(1)[0]
    g = pt.get_gradient()
    _, _, eta, _, _ = pt.get_state()
    dF, bnd = pt.get_ls_partials(with_bound=True)
    dh = d.cpu().numpy()
    pt.close()
    return dict(w=w, p=p.astype(np.complex64).astype(np.complex128), scan=scan, d=dh, u0=u0, tr=tr, g=g, eta=eta,
                dF=dF, bnd=bnd)


def test_farfield_sampled_frames(paper_run):
    r = paper_run
    rng = np.random.default_rng(0)
    idx = rng.choice(len(r["scan"]), 16, replace=False)
    psi0 = np.ones((r["w"].H, r["w"].W), np.complex128)
    ref = O.forward_G(psi0, r["p"], r["scan"][idx])
    got = r["u0"][idx]
    assert np.linalg.norm(got - ref) <= 2e-6 * np.linalg.norm(ref)


def test_gradient_sampled_pixels(paper_run):
    r = paper_run
    scan, p, d, N = r["scan"], r["p"], r["d"], r["w"].N
    rng = np.random.default_rng(1)
    lo, hi = int(scan[:, 0].min()), int(scan[:, 0].max()) + N
    pix = np.stack([rng.integers(lo, hi, 48), rng.integers(lo, hi, 48)], 1)
    pix = np.concatenate([pix, [[lo, lo], [hi - 1, hi - 1], [lo + N // 2, hi - 1]]])
    psi0 = np.ones((r["w"].H, r["w"].W), np.complex128)
    refs, r32s, gots = [], [], []
    p32 = p.astype(np.complex64)
    for (y, x) in pix:
        cov = np.where((scan[:, 0] <= y) & (y < scan[:, 0] + N) & (scan[:, 1] <= x) & (x < scan[:, 1] + N))[0]
        acc, acc32 = 0j, 0j
        for j in cov:
            u = O.ufft2(p * O.extract(psi0, scan[j], N))
            yj = np.conj(p) * O.uifft2(O.residual(u, d[j].astype(np.float64)))
            acc += yj[y - scan[j, 0], x - scan[j, 1]]
            # the same formula in plain float32 (the e32 yardstick of the parity protocol)
            u32 = np.fft.fft2(p32, norm="ortho").astype(np.complex64)
            a2 = (u32.real ** 2 + u32.imag ** 2).astype(np.float32)
            q = np.where(a2 >= np.float32(1e-32), d[j] / np.where(a2 > 0, a2, 1), 0).astype(np.float32)
            y32 = np.conj(p32) * np.fft.ifft2((u32 - q * u32).astype(np.complex64), norm="ortho")
            acc32 += complex(y32[y - scan[j, 0], x - scan[j, 1]])
        refs.append(acc)
        r32s.append(acc32)
        gots.append(complex(r["g"][y, x]))
    refs, r32s, gots = np.array(refs), np.array(r32s), np.array(gots)
    rms = np.sqrt(np.mean(np.abs(refs) ** 2))
    # psi_0 = 1 makes u = F(p) tiny where d > 0 (the residual is ill-conditioned there, SURVEY
    # 8(c).4), so the parity protocol's teacher-forced rule applies over the sample:
    # rel L2 <= max(1e-4, 4 e32), e32 = rel L2 error of the plain float32 evaluation
    e32 = np.linalg.norm(r32s - refs) / np.linalg.norm(refs)
    err = np.linalg.norm(gots - refs) / np.linalg.norm(refs)
    assert err <= max(1e-4, 4 * e32), (err, e32)


def test_first_line_search_all_frames(paper_run):
    r = paper_run
    scan, p, d, N = r["scan"], r["p"], r["d"], r["w"].N
    eta = r["eta"].astype(np.complex128)
    kstar = r["tr"]["shrinks"]
    ks = [k for k in (kstar - 1, kstar) if k >= 0]   # the decision boundary (cost: 2 trials)
    tot = {k: 0.0 for k in ks}
    scale = {k: 0.0 for k in ks}
    psi0 = np.ones((N, N), np.complex128)
    u = O.ufft2(p * psi0)                       # psi_0 = 1: the same far field for every frame
    for a in range(0, len(scan), 2048):
        sc = scan[a:a + 2048]
        v = O.forward_G(eta, p, sc)
        dd = d[a:a + 2048].astype(np.float64)
        uu = np.broadcast_to(u, v.shape)
        for k in ks:
            g = 0.5 ** k
            tot[k] += O.ls_delta(uu, v, dd, g)
            scale[k] += np.sum(np.abs(uu + g * v) ** 2) + np.sum(np.abs(uu) ** 2) + \
                2 * np.sum(np.abs(dd * np.log(np.maximum(np.abs(uu), 1e-30))))
    for k in ks:
        assert abs(r["dF"][k] - tot[k]) <= max(1e-5 * scale[k], 2 * r["bnd"][k]), (k, r["dF"][k], tot[k])
    # the GPU's accepted trial is the oracle's first accepted one (Eq.7 with t = 0)
    assert tot[kstar] <= 0
    if kstar > 0:
        assert tot[kstar - 1] > 0
