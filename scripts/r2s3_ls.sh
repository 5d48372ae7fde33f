#!/bin/bash
# gpurun: k_ls_ws epilogue variants (ping-pong u/d registers; v stored by the FFT group, PTYGER_PF=3)
# against the HEAD build (libptyger_base.so), paper view; parity of the production N = 128 fixtures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3c}
B=PTYGER_LIB=$PWD/paper_2106_07575_b200/libptyger_base.so
for PFV in 1 3; do
  PTYGER_PF=$PFV timeout 900 python -m pytest -m gpu -q -x --timeout=600 tests/test_gpu_production.py -k "n128" > gpurun_out/pytest_${TAG}_pf${PFV}.log 2>&1
  echo "pf=$PFV pytest rc=$?"; tail -1 gpurun_out/pytest_${TAG}_pf${PFV}.log
done
bash scripts/ab_ls.sh $B X=1 PTYGER_PF=3 $B X=1 PTYGER_PF=3
