#!/bin/bash
# gpurun: ncu --set full of the default LS kernels (k_ls_ws at the paper config, k_ls_c256 at the large
# config), a large-view bench line (LS pass counts), and the paper-config default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2d}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls_ws$' -s 2 -c 1 \
    -o gpurun_out/prof_lsws_${TAG} -f $B > gpurun_out/ncu_lsws_${TAG}.log 2>&1
echo "ncu lsws rc=$?" >> gpurun_out/ncu_lsws_${TAG}.log
timeout 900 python bench.py --config large --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/large_${TAG}.json 2> gpurun_out/large_${TAG}.err
BL="python bench.py --config large --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls_c256$' -s 1 -c 1 \
    -o gpurun_out/prof_c256_${TAG} -f $BL > gpurun_out/ncu_c256_${TAG}.log 2>&1
echo "ncu c256 rc=$?" >> gpurun_out/ncu_c256_${TAG}.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-large --e2e-steps 0 --no-cpu-baseline > gpurun_out/paper_${TAG}.json 2> gpurun_out/paper_${TAG}.err
for f in large paper; do python - <<PY
import json
l=[x for x in open('gpurun_out/${f}_${TAG}.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l); r=d['roofline']
print('$f: value %.0f ms %.3f k_ls %.3f k_grad %.3f frac %.3f iter_frac %.3f stage %s shrinks %s passes %s' % (d['value'], d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], r['frac'], d['iteration_roofline']['frac'], {k: round(v,3) for k,v in d['stage_ms'].items()}, d.get('shrinks'), d.get('ls_passes')))
PY
done
tail -1 gpurun_out/ncu_lsws_${TAG}.log gpurun_out/ncu_c256_${TAG}.log
