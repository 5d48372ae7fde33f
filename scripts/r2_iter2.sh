#!/bin/bash
# gpurun: GPU suite (minus the 5-minute large all-frames check), LS A/B, ncu of k_ls_ws, large bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -s --timeout=1500 -k "not large_first_line_search_all_frames" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -n 4 gpurun_out/pytest_${TAG}.log
bash scripts/ab_ls.sh PTYGER_LS_WS=1 > gpurun_out/ab_${TAG}.txt 2>&1
cat gpurun_out/ab_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls_ws$' -s 2 -c 1 \
    -o gpurun_out/prof_lsws_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large > gpurun_out/ncu_lsws_${TAG}.log 2>&1
echo "ncu rc=$?"
