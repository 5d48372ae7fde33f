#!/bin/bash
# gpurun (round 2 evidence): sanitizers of the small fixtures (incl. frames > CTAs), ncu --set full of the
# paper-scale LS kernel, the ncu launch list of a short default bench, the default bench line (paper +
# e2e + CPU baseline + large view), the 3-D batch line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2final}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from tests._common import get_fixture
from paper_2106_07575_b200 import _lib as L
for name in ("tiny", "n64", "n128", "n256", "n128m"):
    psi_true, p, scan, d = get_fixture(name)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    print(name, [t["shrinks"] for t in pt.iterate(3)], flush=True)
    pt.close()
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python /tmp/one.py > gpurun_out/${tool}_${TAG}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tool}_${TAG}.log
done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls_ws|grad|adj)$' -s 3 -c 3 \
    -o gpurun_out/prof_paper_${TAG} -f $B > gpurun_out/ncu_paper_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_paper_${TAG}.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_paper_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 1800 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 900 python bench.py --config view3d --no-cpu-baseline > gpurun_out/view3d_${TAG}.json 2> gpurun_out/view3d_${TAG}.err
echo "view3d rc=$?"
for t in memcheck racecheck synccheck; do tail -n 2 gpurun_out/${t}_${TAG}.log; done
tail -n 1 gpurun_out/ncu_paper_${TAG}.log
