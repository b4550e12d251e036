cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
for lib in paper_2004_02003_b200/liblag.so paper_2004_02003_b200/liblag_pf.so; do
  for cfg in C5 C3; do
    echo "== $lib $cfg"; LAG_LIB=$lib timeout 300 python scripts/time_advect.py $cfg 3 2>&1 | tail -1
  done
done
LAG_LIB=paper_2004_02003_b200/liblag_pf.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
