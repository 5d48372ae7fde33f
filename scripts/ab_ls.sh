#!/bin/bash
# gpurun: k_ls A/B over env settings (each line: VAR=val ...), paper config, 20 timed iterations.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
summ() { python -c "import sys,json; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); r=d['roofline']; print('value %.0f ms %.3f k_ls %.3f k_grad %.3f frac_ls %.3f shrinks %.2f stage %s' % (d['value'], d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], 8314421248/(r['k_ls_avg_ms']*1e-3)/1e9/6454, d['mean_shrinks'], {k: round(v,3) for k,v in d['stage_ms'].items()}))"; }
for SET in "$@"; do
  echo -n "$SET: "; env $SET timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large 2>>gpurun_out/ab.err | summ
done
