#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from tests.test_gpu_parity import get_fixture
from paper_2106_07575_b200 import _lib as L
psi_true, p, scan, d = get_fixture("n128")
pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
print(pt.iterate(3))
PY
PTYGER_LS_V1=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/one.py > gpurun_out/san_grad128.log 2>&1
PTYGER_GRAD_V1=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/one.py > gpurun_out/san_ls128.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v1.log 2>&1
PTYGER_GRAD_V1=1 timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ls128.log 2>&1
tail -30 gpurun_out/san_grad128.log; tail -30 gpurun_out/san_ls128.log; tail -3 gpurun_out/pytest_v1.log; tail -3 gpurun_out/pytest_ls128.log
