#!/bin/bash
# A/B of environment toggles: bash scripts/ab_env.sh TAG "VAR=a" "VAR=b" ...  (bench only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_${TAG}_$i.log 2>&1
  python - "gpurun_out/ab_${TAG}_$i.log" "$e" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[2],"value %.4g"%d["value"],"ms %.3f"%d["ms_per_step"],{k:round(v,3) for k,v in d["stage_ms"].items()},"shrinks",d.get("mean_shrinks"))
PY
  i=$((i+1))
done
