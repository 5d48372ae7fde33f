#!/bin/bash
# A/B of the TMA-ring frame kernels vs the generic ones on the paper config + ncu of each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-ab}
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${TAG}_ring.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${TAG}_v1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_grad128|k_ls128' -s 2 -c 2 \
    -o gpurun_out/prof_${TAG}_ring -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_${TAG}_ring.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_grad|k_ls<' -s 2 -c 2 \
    -o gpurun_out/prof_${TAG}_v1 -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_${TAG}_v1.log 2>&1
for f in gpurun_out/bench_${TAG}_ring.log gpurun_out/bench_${TAG}_v1.log; do python -c "
import json,sys;l=[x for x in open('$f') if x.startswith('{')];d=json.loads(l[0]) if l else {}
print('$f', d.get('value'), d.get('stage_ms'))"; done
tail -2 gpurun_out/ncu_${TAG}_ring.log gpurun_out/ncu_${TAG}_v1.log
