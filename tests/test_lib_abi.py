"""CPU tests of the C ABI boundary (no GPU): the library loads, exports every symbol the
header declares, its host-side partition is bit-exact with the oracle's, and device calls
fail loudly (no CPU fallback) when there is no GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ptyger.h")


@pytest.fixture(scope="module")
def L():
    from paper_2106_07575_b200 import build
    build.build(verbose=False)
    from paper_2106_07575_b200 import _lib
    return _lib


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ptyger_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 17
    for nm in names:
        assert hasattr(L.lib, nm), nm


def test_round_positions_examples(L):
    got = L.round_positions([[2.4, 3.6], [2.5, 3.5], [-0.4, 0.0], [0.49999997, 1.5]])
    assert got.tolist() == [[2, 4], [3, 4], [0, 0], [0, 2]]      # S:75-77 + float32 trap


def test_partition_bit_exact_with_oracle(L):
    from oracle import partition as Pt
    from paper_2106_07575_b200 import inputs as I
    rng = np.random.default_rng(11)
    cases = []
    for name in ("tiny", "mid"):
        w = I.WORKLOADS[name]
        cases.append((I.workload_inputs(w)[2], w.H, w.N))
    for _ in range(15):
        H, N = 200, 16
        n = int(rng.integers(10, 150))
        cases.append((np.stack([rng.integers(0, H - N + 1, n), rng.integers(0, H - N + 1, n)], 1), H, N))
    checked = 0
    for scan, H, N in cases:
        for P in range(1, 9):
            if not Pt.feasible(scan, N, P):
                with pytest.raises(L.PtygerError) as ei:
                    L.partition(scan, H, N, P)
                assert ei.value.status == 2 and "largest feasible P = %d" % Pt.max_feasible_P(scan, N) in str(ei.value)
                continue
            rk, rows = L.partition(scan, H, N, P)
            ork, orows = Pt.partition(scan, H, N, P)
            assert np.array_equal(rk, ork)
            assert np.array_equal(rows, np.array(orows, dtype=np.int64))
            checked += 1
    assert checked > 30


def test_partition_rejects_out_of_bounds(L):
    with pytest.raises(L.PtygerError) as ei:
        L.partition(np.array([[0, 0], [60, 0]]), 64, 16, 1)
    assert ei.value.status == 3 and "frame 1" in str(ei.value)


def test_device_calls_fail_loudly_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_07575_b200 import inputs as I
    w = I.WORKLOADS["tiny"]
    psi, p, scan = I.workload_inputs(w)
    d = np.ones((len(scan), 16, 16), np.float32)
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(np.ones_like(psi), p, scan, d)
    assert ei.value.status == 5 and "no CUDA device" in str(ei.value)


def test_init_validation_before_device(L):
    from paper_2106_07575_b200 import inputs as I
    w = I.WORKLOADS["tiny"]
    psi, p, scan = I.workload_inputs(w)
    d = np.ones((len(scan), 16, 16), np.float32)
    bad = scan.copy()
    bad[7] = [60, 0]
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(psi, p, bad, d)
    assert ei.value.status == 3 and "frame 7" in str(ei.value)
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(psi, p, scan, d, ls_batch=17)
    assert ei.value.status == 2
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(np.ones((64, 64), complex), np.ones((24, 24), complex), scan, np.ones((len(scan), 24, 24), np.float32))
    assert ei.value.status == 2
    # intensities that do not hold n*N*N values are rejected before any pointer reaches the library
    with pytest.raises(L.PtygerError) as ei:
        L.Ptyger(psi, p, scan, d[:-1])
    assert ei.value.status == 3 and "n*N*N" in str(ei.value)


def test_header_documents_boundary():
    src = open(HEADER).read()
    for cite in ["PAPER.md:411-415", "PAPER.md:426-430", "PAPER.md:432-436", "PAPER.md:447-453", "PAPER.md:454-460"]:
        assert cite in src
