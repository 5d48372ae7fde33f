#!/bin/bash
# gpurun: k_ls A/B (warp-specialised k_ls_ws vs single-group k_ls<128>) + quick N=128 parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-ab}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
summ() { python -c "import sys,json; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); r=d['roofline']; print('value %.0f ms %.3f k_ls %.3f k_grad %.3f frac_ls %.3f shrinks %.2f stage %s' % (d['value'], d['ms_per_step'], r['k_ls_avg_ms'], r['k_grad_avg_ms'], 8314421248/(r['k_ls_avg_ms']*1e-3)/1e9/6454, d['mean_shrinks'], d['stage_ms']))"; }
for WS in 1 0 1; do
  echo -n "WS=$WS: "; PTYGER_LS_WS=$WS timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large 2>gpurun_out/ab_${TAG}_${WS}.err | summ
done
timeout 900 python -m pytest -m gpu -q -x --timeout=600 -k "n128 or tiny or fft or kernel_timers or single_frame or subpixel" tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_subpixel.py 2>&1 | tail -5
