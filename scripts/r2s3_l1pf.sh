#!/bin/bash
# gpurun: k_ls_ws epilogue L1 prefetch three groups ahead (PTYGER_PF bit 2) against the HEAD build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
B=PTYGER_LIB=$PWD/paper_2106_07575_b200/libptyger_base.so
PTYGER_PF=5 timeout 900 python -m pytest -m gpu -q -x --timeout=600 tests/test_gpu_production.py -k "n128m and not schedule" > gpurun_out/pytest_l1pf.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_l1pf.log
bash scripts/ab_ls.sh $B PTYGER_PF=1 PTYGER_PF=5 PTYGER_PF=4 $B PTYGER_PF=1 PTYGER_PF=5 PTYGER_PF=4
