#!/bin/bash
# gpurun: one `ncu --set full --import-source on` capture each of k_ls<128> and k_grad128 at the
# paper config (3rd launch of each, after warm-up), plus the launch list of a short bench run.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r1e}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls(_hf)?$' -s 2 -c 1 \
    -o gpurun_out/prof_ls_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_ls_${TAG}.log 2>&1
echo "ncu ls rc=$?" >> gpurun_out/ncu_ls_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_grad(128|_hf)?$' -s 2 -c 1 \
    -o gpurun_out/prof_grad_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_grad_${TAG}.log 2>&1
echo "ncu grad rc=$?" >> gpurun_out/ncu_grad_${TAG}.log
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch_${TAG}.log
fi
tail -2 gpurun_out/ncu_ls_${TAG}.log; tail -2 gpurun_out/ncu_grad_${TAG}.log
