#!/bin/bash
# gpurun (round 2): source-level ncu capture of the LS and GRAD frame kernels at the paper config,
# compute-sanitizer memcheck / racecheck of a small config, ncu launch list of a short bench run.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r2a}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KRE=${KRE:-'regex:^k_ls$'}
timeout 900 ncu --set full --clock-control none --import-source on -k "$KRE" -s 2 -c 1 \
    -o gpurun_out/prof_ls_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_ls_${TAG}.log 2>&1
echo "ncu ls rc=$?" >> gpurun_out/ncu_ls_${TAG}.log
if [ -n "$SANITIZE" ]; then
cat > /tmp/one.py <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from tests.test_gpu_parity import get_fixture
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
fi
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch_${TAG}.log
fi
tail -2 gpurun_out/ncu_ls_${TAG}.log; tail -3 gpurun_out/memcheck_${TAG}.log 2>/dev/null; tail -3 gpurun_out/racecheck_${TAG}.log 2>/dev/null
