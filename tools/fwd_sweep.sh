#!/bin/bash
# Forward-kernel variant sweep (kernel_times.py under different CTIS_FWD_* settings).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-sweep}_fwd_sweep.txt
: > $OUT
for cfg in ${CFGS:-C4 C3}; do
  for v in "2 32" "2 18" "3 24" "3 18" "3 14" "4 16" "4 14" "4 10"; do
    set -- $v
    CTIS_FWD_OCC=$1 CTIS_FWD_MAXM=$2 timeout 120 python tools/kernel_times.py $cfg 2>&1 | sed "s/^/occ$1 cap$2 /" >> $OUT
  done
done
