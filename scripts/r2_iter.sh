#!/bin/bash
# gpurun: GPU suite (minus the 5-minute large all-frames check unless FULL=1), LS-kernel A/B at the
# paper config, a short large-view bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
SEL="not large_first_line_search_all_frames"
[ -n "$FULL" ] && SEL=""
timeout 2400 python -m pytest tests -m gpu -q -x -s --timeout=1500 -k "$SEL" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -5 gpurun_out/pytest_${TAG}.log
bash scripts/ab_ls.sh PTYGER_LS_WS=1 PTYGER_LS_WS=0 > gpurun_out/ab_${TAG}.txt 2>&1
cat gpurun_out/ab_${TAG}.txt
timeout 900 python bench.py --config large --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/large_${TAG}.json 2> gpurun_out/large_${TAG}.err
python - <<PY
import json
l=[x for x in open('gpurun_out/large_${TAG}.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l); r=d['roofline']
print('large: value %.0f ms %.2f k_ls %.2f k_grad %.2f iter_frac %.3f stage %s shrinks %s' % (d['value'], d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], d['iteration_roofline']['frac'], {k: round(v,2) for k,v in d['stage_ms'].items()}, d.get('mean_shrinks')))
PY
