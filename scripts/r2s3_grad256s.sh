#!/bin/bash
# gpurun (round 2, session 3): parity of the staged N = 256 GRAD kernel (k_grad256s) at the production
# fixtures, large-view A/B staged vs synchronous k_grad256, one ncu --set full capture of each, and a
# source-level capture of the paper-scale k_ls_ws.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest -m gpu -q -x -s --timeout=900 tests/test_gpu_production.py -k "n256" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
grep -q "pytest rc=0" gpurun_out/pytest_${TAG}.log || exit 1
bash scripts/ab_large.sh PTYGER_GRAD256_STAGE=0 PTYGER_GRAD256_STAGE=1 PTYGER_GRAD256_STAGE=0 PTYGER_GRAD256_STAGE=1
for S in 0 1; do
  PTYGER_GRAD256_STAGE=$S timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_grad256s?$' -s 2 -c 1 \
    -o gpurun_out/prof_g256_${S}_${TAG} -f python bench.py --config large --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_g256_${S}_${TAG}.log 2>&1
  echo "ncu g256 $S rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls_ws$' -s 3 -c 1 \
    -o gpurun_out/prof_lsws_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large \
    > gpurun_out/ncu_lsws_${TAG}.log 2>&1
echo "ncu lsws rc=$?"
