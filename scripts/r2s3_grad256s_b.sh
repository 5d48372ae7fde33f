#!/bin/bash
# gpurun: staged k_grad256s (pass-1 staging only) parity at the N = 256 production fixtures + large A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest -m gpu -q -x -s --timeout=900 tests/test_gpu_production.py -k "n256m" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -2 gpurun_out/pytest_${TAG}.log
bash scripts/ab_large.sh PTYGER_GRAD256_STAGE=0 PTYGER_GRAD256_STAGE=1 PTYGER_GRAD256_STAGE=1
PTYGER_GRAD256_STAGE=1 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_grad256s?$' -s 2 -c 1 \
    -o gpurun_out/prof_g256_1_${TAG} -f python bench.py --config large --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_g256_1_${TAG}.log 2>&1
echo "ncu rc=$?"
