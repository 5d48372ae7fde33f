#!/bin/bash
# gpurun: selected GPU test files with their printed diagnostics (-s) and per-test durations.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-t}
shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 3000 python -m pytest -m gpu -q -s --timeout=1500 --durations=15 "$@" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -30 gpurun_out/pytest_${TAG}.log
