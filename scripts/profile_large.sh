#!/bin/bash
# gpurun: one `ncu --set full` capture each of the N = 256 frame kernels (large config, 2nd iteration).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-large}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls_c256|grad256)$' -s 2 -c 2 \
    -o gpurun_out/prof_${TAG} -f python bench.py --config l256p --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_${TAG}.log
tail -3 gpurun_out/ncu_${TAG}.log
