#!/bin/bash
# gpurun: parity tests (subset), bench, ncu launch list + full capture of the hot kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_ls|k_grad|k_adj' -c 3 \
    -o gpurun_out/prof_${TAG} -f python bench.py --config small --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/smoke.log; tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log; tail -3 gpurun_out/ncu_full.log
