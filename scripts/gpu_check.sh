#!/bin/bash
# One gpurun call: smoke, GPU tests (per-test timeout), bench.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-chk}
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=300 ${PYTEST_K} > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
tail -2 gpurun_out/smoke.log; tail -4 gpurun_out/pytest_gpu_${TAG}.log; tail -2 gpurun_out/bench_${TAG}.log | cut -c1-400
