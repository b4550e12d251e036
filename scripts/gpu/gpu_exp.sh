#!/bin/bash
# kernel experiment: time library variants (C5, C3) and run parity against one
# usage: gpu_exp.sh "<lib suffixes>" <parity suffix>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
for v in $1; do
  lib=paper_2004_02003_b200/liblag${v:+_$v}.so
  [ "$v" = "base" ] && lib=paper_2004_02003_b200/liblag.so
  for cfg in C5 C3; do
    echo "== $v $cfg"; LAG_LIB=$lib timeout 300 python scripts/time_advect.py $cfg 3 2>&1 | tail -1
  done
done
if [ -n "$2" ]; then
  LAG_LIB=paper_2004_02003_b200/liblag_$2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -3
fi
