#!/bin/bash
# gpurun: 8-entry trial-sum reduce-scatter for passes of <= 8 trials (LS pass-0 kernels) against HEAD.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B=PTYGER_LIB=$PWD/paper_2106_07575_b200/libptyger_base.so
timeout 1200 python -m pytest -m gpu -q -x --timeout=900 tests/test_gpu_production.py tests/test_gpu_parity.py -k "teacher or trajectory or schedule" > gpurun_out/pytest_kr.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_kr.log
bash scripts/ab_ls.sh $B X=1 $B X=1
bash scripts/ab_large.sh $B X=1
