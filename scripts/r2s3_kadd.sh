#!/bin/bash
# gpurun: margin of the adaptive pass-0 trial count (keff = k*_prev + PTYGER_KEFF_ADD) at both views.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash scripts/ab_large.sh PTYGER_KEFF_ADD=3 PTYGER_KEFF_ADD=4 PTYGER_KEFF_ADD=5 PTYGER_KEFF_ADD=6
bash scripts/ab_ls.sh PTYGER_KEFF_ADD=3 PTYGER_KEFF_ADD=4 PTYGER_KEFF_ADD=5
