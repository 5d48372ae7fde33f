#!/bin/bash
# gpurun: sparse-aware k_lsx (u, v read only where d > 0 under the object-grid q part): parity + large view.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_lsx.log 2>&1 || { tail gpurun_out/build_lsx.log; exit 1; }
timeout 1500 python -m pytest -m gpu -q -x --timeout=900 tests/test_gpu_parity.py tests/test_gpu_production.py \
    tests/test_gpu_fullsize.py > gpurun_out/pytest_lsx.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lsx.log
bash scripts/ab_large.sh X=1 X=1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:^k_lsx$' --csv \
    --log-file gpurun_out/lsx_launches.csv python bench.py --config large --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo "ncu rc=$?"
