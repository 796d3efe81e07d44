#!/bin/bash
# ncu --set full of the pair-local PCDM kernels at C2 (second solve of configs.py: warm)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cd_pair_kernel|mt_words_kernel|cd_prevd_kernel" -s 3 -c 3 -o gpurun_out/pcdm_pair python configs.py --only c2 --no-cpu > gpurun_out/pcdm_pair_prof.log 2>&1
echo "exit $?" >> gpurun_out/pcdm_pair_prof.log
