#!/bin/bash
# gpurun: conj(p / N) applied by k_adj instead of the GRAD frame kernels (PTYGER_ADJ_PROBE=1): parity of the
# teacher-forced / subpixel / production tests in that mode, A/B at both views.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_adjp.log 2>&1 || { tail gpurun_out/build_adjp.log; exit 1; }
PTYGER_ADJ_PROBE=1 timeout 1500 python -m pytest -m gpu -q -x --timeout=900 tests/test_gpu_parity.py tests/test_gpu_subpixel.py \
    tests/test_gpu_production.py -k "not schedule" > gpurun_out/pytest_adjp.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_adjp.log
bash scripts/ab_ls.sh PTYGER_ADJ_PROBE=0 PTYGER_ADJ_PROBE=1 PTYGER_ADJ_PROBE=0 PTYGER_ADJ_PROBE=1
bash scripts/ab_large.sh PTYGER_ADJ_PROBE=0 PTYGER_ADJ_PROBE=1 PTYGER_ADJ_PROBE=0 PTYGER_ADJ_PROBE=1
