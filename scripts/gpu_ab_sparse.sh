#!/bin/bash
# A/B of libl1b builds on the CSR/CSC (north-star) FISTA leg.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LIB=paper_1503_03520_b200/lib/libl1b.so
cp $LIB abtest/libl1b_keep.so
for round in 1 2; do
  for v in ${AB_VARIANTS:-old new}; do
    cp abtest/libl1b_$v.so $LIB
    echo "== $v" >> gpurun_out/ab_sparse.log
    timeout 900 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); sp=d['sparse_path']
        print('sparse', round(sp['value'],2), 'k1', round(sp['kernels_ms']['fista_k1'],3), 'k2', round(sp['kernels_ms']['fista_k2'],3), 'gbs', round(sp['hbm_gbs_ax_atr'],1), 'mf', round(d['value'],1))
" >> gpurun_out/ab_sparse.log
  done
done
cp abtest/libl1b_keep.so $LIB
