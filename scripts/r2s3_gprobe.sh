#!/bin/bash
# gpurun: k_grad256 with half of its probe columns resident in shared memory, against HEAD.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B=PTYGER_LIB=$PWD/paper_2106_07575_b200/libptyger_base.so
timeout 1200 python -m pytest -m gpu -q -x --timeout=900 tests/test_gpu_production.py tests/test_gpu_parity.py -k "n256" > gpurun_out/pytest_gp.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gp.log
bash scripts/ab_large.sh $B X=1 $B X=1
