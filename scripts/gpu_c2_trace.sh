#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L1B_PCDM_TRACE=1 timeout 600 python configs.py --only c2 --no-cpu > gpurun_out/c2_trace.log 2>&1; echo "exit $?" >> gpurun_out/c2_trace.log
