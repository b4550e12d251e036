cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
L=paper_2004_02003_b200
for c in C5 C3; do
echo "== base $c"; timeout 300 python scripts/time_advect.py $c 3 2>&1 | tail -1
echo "== node $c"; LAG_LIB=$L/liblag_node.so timeout 300 python scripts/time_advect.py $c 3 2>&1 | tail -1
done
LAG_LIB=$L/liblag_node.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
