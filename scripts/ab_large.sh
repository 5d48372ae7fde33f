#!/bin/bash
# gpurun: large-view A/B over env settings (each argument: VAR=val ...), LSTEPS (default 10) timed iterations after 3 warm-up.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for SET in "$@"; do
  echo -n "$SET: "
  env $SET timeout 900 python bench.py --config large --steps ${LSTEPS:-10} --warmup 3 --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/ab_large.err | python -c "
import sys, json
d = json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); r = d['roofline']
print('ms %.2f k_ls %.2f k_grad %.2f iter_frac %.3f stage %s shrinks %s passes %s' % (d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], d['iteration_roofline']['frac'], {k: round(v, 2) for k, v in d['stage_ms'].items()}, d.get('shrinks'), d.get('ls_passes')))"
done
