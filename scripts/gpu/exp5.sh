cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
echo "== brick"; LAG_BRICK=1 timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -3
echo "== old"; timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -15
