#!/bin/bash
# gpurun: sparse-aware k_lsx with the next batch's d prefetched, against HEAD: ncu time + DRAM bytes of the
# large view's extra LS pass, parity, large-view A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B=$PWD/paper_2106_07575_b200/libptyger_base.so
for L in new base; do
  if [ $L = base ]; then export PTYGER_LIB=$B; else unset PTYGER_LIB; fi
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k 'regex:^k_lsx$' --csv \
      --log-file gpurun_out/lsx2_${L}.csv python bench.py --config large --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  echo "ncu $L rc=$?"
done
unset PTYGER_LIB
timeout 1500 python -m pytest -m gpu -q -x --timeout=900 tests/test_gpu_parity.py tests/test_gpu_production.py > gpurun_out/pytest_lsx2.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lsx2.log
bash scripts/ab_large.sh PTYGER_LIB=$B X=1 PTYGER_LIB=$B X=1
