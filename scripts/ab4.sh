#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout=200 -k "teacher and n128" > gpurun_out/ab4_pytest.log 2>&1
for rep in 1 2; do
  timeout 300 $B > gpurun_out/ab4_ring_$rep.log 2>&1
  PTYGER_GRAD_V1=1 timeout 300 $B > gpurun_out/ab4_v1_$rep.log 2>&1
done
PTYGER_LS_RING=1 timeout 300 $B > gpurun_out/ab4_lsring.log 2>&1
tail -2 gpurun_out/ab4_pytest.log
for f in ring_1 v1_1 ring_2 v1_2 lsring; do python -c "
import json;l=[x for x in open('gpurun_out/ab4_$f.log') if x.startswith('{')];d=json.loads(l[0]) if l else {}
s=d.get('stage_ms',{}); print('$f', round(d.get('value',0)), {k: round(v,3) for k,v in s.items()}, d.get('mean_shrinks'), d.get('clocks',{}).get('sm_mhz'))"; done
