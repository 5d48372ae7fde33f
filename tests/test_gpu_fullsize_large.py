"""Parity at BASELINE.json's large view (8192^2 object, 256^2 detector, 99 856 frames) on one GPU, in the
launch configuration bench.py times (cluster-of-four LS kernel, v-slot GRAD kernel), from a
WELL-CONDITIONED state (I.conditioned_state), on outputs the float64 oracle can compute one by one,
plus properties that hold at any size:

* grad F at sampled object pixels after the first iteration, each recomputed by the oracle on the
  sub-problem of only the frames covering it; e32 of the sample asserted < 2.5e-5, so the bar is 1e-4;
* the first iteration's DeltaF_k at the decision boundary (k*-1, k*) over ALL 99 856 frames (oracle far
  fields chunked, scipy.fft threads): within 1e-5 sum|terms|, the GPU's accepted trial is the first
  accepted one;
* the first iterations decrease F (Eq.7 with t = 0), every gamma is a trial of gamma_0 tau^k.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_gpu_fullsize import boundary_deltas, run_view, sampled_gradient  # noqa: E402


@pytest.fixture(scope="module")
def large_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if torch.cuda.get_device_properties(0).total_memory < 170e9:
        pytest.skip("large view needs ~160 GB of device memory")
    return run_view("large", iters_after=2)


def test_large_gradient_sampled_pixels(large_run):
    r = large_run
    scan, N = r["scan"], r["w"].N
    rng = np.random.default_rng(2)
    lo, hi = int(scan[:, 0].min()), int(scan[:, 0].max()) + N
    pix = np.stack([rng.integers(lo, hi, 10), rng.integers(lo, hi, 10)], 1)
    pix = np.concatenate([pix, [[lo, lo], [hi - 1, hi - 1]]])
    gots, refs, r32s = sampled_gradient(r, pix)
    e32 = np.linalg.norm(r32s - refs) / np.linalg.norm(refs)
    err = np.linalg.norm(gots - refs) / np.linalg.norm(refs)
    print(f"large: sampled gradient err {err:.2e}, e32 {e32:.2e}")
    assert e32 < 2.5e-5, e32
    assert err <= 1e-4, (err, e32)


def test_large_first_line_search_all_frames(large_run):
    r = large_run
    kstar = r["tr"]["shrinks"]
    assert not r["tr"]["stalled"] and len(r["dF"]) == kstar + 1
    ks = [k for k in (kstar - 1, kstar) if k >= 0]
    tot, scale = boundary_deltas(r, ks, chunk=512)
    for k in ks:
        print(f"large: DeltaF_{k} gpu {r['dF'][k]:.9e} oracle {tot[k]:.9e} (rel to scale "
              f"{abs(r['dF'][k] - tot[k]) / scale[k]:.1e})")
        assert abs(r["dF"][k] - tot[k]) <= 1e-5 * scale[k], (k, r["dF"][k], tot[k], scale[k])
    assert tot[kstar] <= 0
    if kstar > 0:
        assert tot[kstar - 1] > 0


def test_large_line_search_properties(large_run):
    trs, F = large_run["trs"], large_run["F0"]
    for t in trs:
        assert not t["stalled"] and t["shrinks"] >= 0
        assert t["gamma"] == 0.5 ** t["shrinks"]
        assert t["F"] <= F            # Eq.7 with t = 0: accepted trials never increase F
        F = t["F"]
    assert trs[-1]["F"] < large_run["F0"]
