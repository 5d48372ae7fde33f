#!/bin/bash
# gpurun: full GPU suite (diagnostics printed), LS-kernel A/B, default bench line (paper + large sub-record).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_${TAG}.txt
timeout 2400 python -m pytest tests -m gpu -q -s --timeout=1500 --durations=25 > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -40 gpurun_out/pytest_${TAG}.log
bash scripts/ab_ls.sh PTYGER_LS_WS=1 PTYGER_LS_WS=0 > gpurun_out/ab_${TAG}.txt 2>&1
cat gpurun_out/ab_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_${TAG}.json
