#!/bin/bash
# gpurun: N = 256 parity (incl. frames > clusters) with the warp-specialised cluster LS kernel, then a
# large-view A/B against the single-group cluster kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-c256}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -s --timeout=900 -k "n256 or s256 or large_gradient or large_line_search_properties" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -n 4 gpurun_out/pytest_${TAG}.log
for V in 1 0; do
PTYGER_C256_WS=$V timeout 900 python bench.py --config large --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/large_${TAG}_$V.json 2> gpurun_out/large_${TAG}_$V.err
python - <<PY
import json
l=[x for x in open('gpurun_out/large_${TAG}_$V.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l); r=d['roofline']
print('WS=$V large: value %.0f ms %.2f k_ls %.2f k_grad %.2f iter_frac %.3f stage %s shrinks %s passes %s' % (d['value'], d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], d['iteration_roofline']['frac'], {k: round(v,2) for k,v in d['stage_ms'].items()}, d.get('shrinks'), d.get('ls_passes')))
PY
done
