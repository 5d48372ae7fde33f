#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/ab3_ring.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 timeout 300 $B > gpurun_out/ab3_v1.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 PTYGER_LS_SPLIT=1 timeout 300 $B > gpurun_out/ab3_split.log 2>&1
PTYGER_GRAD_V1=1 PTYGER_LS_V1=1 PTYGER_LS_SPLIT=1 timeout 600 ncu --set full --clock-control none -k 'regex:k_lsx|k_fwd' -s 3 -c 3 -o gpurun_out/prof_ab3_split -f $B --steps 1 --warmup 1 > gpurun_out/ncu_ab3.log 2>&1
for f in ring v1 split; do python -c "
import json;l=[x for x in open('gpurun_out/ab3_$f.log') if x.startswith('{')];d=json.loads(l[0]) if l else {}
print('$f', d.get('value'), d.get('stage_ms'), d.get('mean_shrinks'))"; done
