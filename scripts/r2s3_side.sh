#!/bin/bash
# gpurun: N = 256 LS side kernel on the SMs the four-CTA clusters leave idle (PDL-released, static tail
# share PTYGER_C256_SIDE per mille): parity at the n256m production fixture, large-view A/B over the share.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python -m pytest -m gpu -q -x -s --timeout=600 tests/test_gpu_production.py -k "n256m" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -12 gpurun_out/pytest_${TAG}.log
grep -q "pytest rc=0" gpurun_out/pytest_${TAG}.log || exit 1
bash scripts/ab_large.sh PTYGER_C256_SIDE=0 PTYGER_C256_SIDE=80 PTYGER_C256_SIDE=100 PTYGER_C256_SIDE=120 PTYGER_C256_SIDE=140 PTYGER_C256_SIDE=0
