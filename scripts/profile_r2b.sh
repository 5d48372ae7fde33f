#!/bin/bash
# gpurun (round 2): ncu --set full of the LS kernels (warp-specialised default and the single-group
# k_ls<128>) at the paper config and of k_ls_c256 / k_grad256 at the large config; memcheck and
# racecheck of the small fixtures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2b}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls_ws$' -s 2 -c 1 \
    -o gpurun_out/prof_lsws_${TAG} -f $B > gpurun_out/ncu_lsws_${TAG}.log 2>&1
echo "ncu lsws rc=$?" >> gpurun_out/ncu_lsws_${TAG}.log
PTYGER_LS_WS=0 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_ls$' -s 2 -c 1 \
    -o gpurun_out/prof_ls_${TAG} -f $B > gpurun_out/ncu_ls_${TAG}.log 2>&1
echo "ncu ls rc=$?" >> gpurun_out/ncu_ls_${TAG}.log
BL="python bench.py --config large --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^k_(ls_c256|grad256)$' -s 2 -c 2 \
    -o gpurun_out/prof_large_${TAG} -f $BL > gpurun_out/ncu_large_${TAG}.log 2>&1
echo "ncu large rc=$?" >> gpurun_out/ncu_large_${TAG}.log
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from tests._common import get_fixture
from paper_2106_07575_b200 import _lib as L
for name in ("tiny", "n64", "n128", "n256"):
    psi_true, p, scan, d = get_fixture(name)
    pt = L.Ptyger(np.ones_like(psi_true), p, scan, d)
    print(name, [t["shrinks"] for t in pt.iterate(3)], flush=True)
    pt.close()
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/one.py > gpurun_out/memcheck_${TAG}.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck_${TAG}.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python /tmp/one.py > gpurun_out/racecheck_${TAG}.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/racecheck_${TAG}.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python /tmp/one.py > gpurun_out/synccheck_${TAG}.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/synccheck_${TAG}.log
for f in ncu_lsws ncu_ls ncu_large memcheck racecheck synccheck; do echo "== $f"; tail -3 gpurun_out/${f}_${TAG}.log; done
