#!/bin/bash
# gpurun: k_grad256b (pass-1 u / slot rows by TMA bulk stores, PTYGER_GRAD256_BULK=1) parity at the n256m
# production fixture and large-view A/B against k_grad256.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
PTYGER_GRAD256_BULK=1 timeout 900 python -m pytest -m gpu -q -x --timeout=600 tests/test_gpu_production.py -k "n256" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -2 gpurun_out/pytest_${TAG}.log
grep -q "pytest rc=0" gpurun_out/pytest_${TAG}.log || exit 1
bash scripts/ab_large.sh PTYGER_GRAD256_BULK=0 PTYGER_GRAD256_BULK=1 PTYGER_GRAD256_BULK=0 PTYGER_GRAD256_BULK=1
PTYGER_GRAD256_BULK=1 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_grad256b$' -s 2 -c 1 \
    -o gpurun_out/prof_g256b_${TAG} -f python bench.py --config large --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_g256b_${TAG}.log 2>&1
echo "ncu rc=$?"
