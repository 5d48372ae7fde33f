#!/bin/bash
# gpurun: bench (paper config), the ncu launch list of a short bench run, and one
# `ncu --set full` capture each of k_grad and k_ls (4th iteration).  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls|grad)$' -s 6 -c 2 \
    -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG}.log
tail -2 gpurun_out/bench_${TAG}.log | cut -c1-300; tail -2 gpurun_out/ncu_launch_${TAG}.log; tail -3 gpurun_out/ncu_full_${TAG}.log
