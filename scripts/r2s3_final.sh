#!/bin/bash
# gpurun (round 2, session 3 evidence): full GPU suite, sanitizers of the small fixtures incl. n256m (the
# N = 256 side kernel and the PDL release), ncu --set full of the paper-scale and large-view frame
# kernels, ncu launch lists of both views, the default bench line (paper + e2e + CPU baseline + large view)
# and the 3-D batch line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
timeout 2400 python -m pytest -m gpu -q -s --timeout=1500 --durations=10 tests > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 900 python bench.py --config view3d --no-cpu-baseline > gpurun_out/view3d_${TAG}.json 2> gpurun_out/view3d_${TAG}.err
echo "view3d rc=$?"
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from tests._common import get_fixture
from paper_2106_07575_b200 import _lib as L
for name in sys.argv[1:]:
    psi_true, p, scan, d = get_fixture(name)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    print(name, [t["shrinks"] for t in pt.iterate(3)], flush=True)
    pt.close()
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python /tmp/one.py tiny n128m n256m > gpurun_out/${tool}_${TAG}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tool}_${TAG}.log
  tail -n 2 gpurun_out/${tool}_${TAG}.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls_ws|grad|adj)$' -s 3 -c 3 \
    -o gpurun_out/prof_paper_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large \
    > gpurun_out/ncu_paper_${TAG}.log 2>&1
echo "ncu paper rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls_c256ws|ls256_side|grad256)$' -s 3 -c 3 \
    -o gpurun_out/prof_large_${TAG} -f python bench.py --config large --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_large_${TAG}.log 2>&1
echo "ncu large rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_paper_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large > gpurun_out/ncu_lp_${TAG}.log 2>&1
echo "launch paper rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_large_${TAG}.csv \
    python bench.py --config large --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_ll_${TAG}.log 2>&1
echo "launch large rc=$?"
