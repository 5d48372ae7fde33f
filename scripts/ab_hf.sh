#!/bin/bash
# A/B of the half-frame cluster kernels (PTYGER_HF=1, default) against the single-CTA path.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-hf}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 ${PYTEST_K} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
for hf in 1 0; do
  PTYGER_HF=$hf timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${TAG}_hf${hf}.log 2>&1
  echo "bench hf=$hf rc=$?" >> gpurun_out/bench_${TAG}_hf${hf}.log
done
tail -3 gpurun_out/pytest_${TAG}.log
for hf in 1 0; do python - "$TAG" "$hf" <<'PY'
import json,sys
tag,hf=sys.argv[1],sys.argv[2]
for l in open(f"gpurun_out/bench_{tag}_hf{hf}.log"):
    if l.startswith("{"):
        d=json.loads(l); print("hf",hf,"value %.4g"%d["value"],"ms %.3f"%d["ms_per_step"],{k:round(v,3) for k,v in d["stage_ms"].items()},"shrinks",d.get("mean_shrinks"))
PY
done
