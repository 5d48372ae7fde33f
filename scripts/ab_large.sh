#!/bin/bash
# A/B of library variants / env toggles on the large config: bash scripts/ab_large.sh TAG "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
i=0
for e in "$@"; do
  env $e timeout 600 python bench.py --config ${CONFIG:-large} --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abl_${TAG}_$i.log 2>&1
  python - "gpurun_out/abl_${TAG}_$i.log" "$e" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[2],"value %.4g"%d["value"],"ms %.3f"%d["ms_per_step"],{k:round(v,3) for k,v in d["stage_ms"].items()},"shrinks",d.get("mean_shrinks"))
PY
  i=$((i+1))
done
