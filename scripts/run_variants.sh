cd "${GRAFT_REPO_ROOT:-/root/repo}"
LAG_LIB=paper_2004_02003_b200/liblag_debug.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/dbg.log 2>&1; echo "debug-bounds pytest exit $?"
grep -E "passed|failed|FAILED|rror" gpurun_out/dbg.log | head -10
