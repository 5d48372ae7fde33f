#!/bin/bash
# gpurun: ncu launch lists (gpu__time_duration, serialised) of short paper and large bench runs, and
# ncu --set full of k_grad256 and the k_lsx screening pass at the large view.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2j}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_paper_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large > gpurun_out/ncu_lp_${TAG}.log 2>&1
echo "launch paper rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_large_${TAG}.csv \
    python bench.py --config large --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_ll_${TAG}.log 2>&1
echo "launch large rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_(grad256|lsx)$' -s 1 -c 2 \
    -o gpurun_out/prof_large2_${TAG} -f python bench.py --config large --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_large2_${TAG}.log 2>&1
echo "ncu large rc=$?"
