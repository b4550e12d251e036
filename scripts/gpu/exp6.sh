cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
L=paper_2004_02003_b200
echo "== base"; timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -1
echo "== adv2 minb3"; LAG_ADV2=1 timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -1
echo "== adv2 minb2"; LAG_ADV2=1 LAG_LIB=$L/liblag_a2m2.so timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -1
echo "== adv2 minb3 C3"; LAG_ADV2=1 timeout 300 python scripts/time_advect.py C3 2 2>&1 | tail -1
echo "== adv2 minb2 C3"; LAG_ADV2=1 LAG_LIB=$L/liblag_a2m2.so timeout 300 python scripts/time_advect.py C3 2 2>&1 | tail -1
LAG_ADV2=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
