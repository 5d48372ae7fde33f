#!/bin/bash
# gpurun: smoke, parity tests, memcheck of the TMA kernels, bench, ncu launch list + full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_parity import get_fixture
from paper_2106_07575_b200 import _lib as L
psi_true, p, scan, d = get_fixture("n128")
pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
print([t["shrinks"] for t in pt.iterate(3)])
PY
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/one.py > gpurun_out/memcheck_${TAG}.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python /tmp/one.py > gpurun_out/racecheck_${TAG}.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_ls|k_grad|k_adj' -s 3 -c 3 \
    -o gpurun_out/prof_${TAG} -f python bench.py --config small --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log; tail -4 gpurun_out/memcheck_${TAG}.log; tail -4 gpurun_out/racecheck_${TAG}.log; tail -2 gpurun_out/bench_${TAG}.log; tail -2 gpurun_out/ncu_full.log
