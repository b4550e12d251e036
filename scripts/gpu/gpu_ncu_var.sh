#!/bin/bash
# full ncu capture of one advect launch (C5, mid-interval) for a library variant
# usage: gpu_ncu_var.sh <suffix> [config]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
v=$1; cfg=${2:-C5}
lib=paper_2004_02003_b200/liblag_$v.so
[ "$v" = "base" ] && lib=paper_2004_02003_b200/liblag.so
LAG_LIB=$lib timeout 300 python scripts/profile_advect.py $cfg 20 > gpurun_out/prof_plain_$v.log 2>&1 || { echo plain failed; tail gpurun_out/prof_plain_$v.log; exit 1; }
LAG_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:advect -s 15 -c 1 \
  -f -o gpurun_out/prof_${v}_$cfg python scripts/profile_advect.py $cfg 20 > gpurun_out/ncu_$v.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_$v.log
