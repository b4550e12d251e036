cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
LAG_LIB= timeout 120 python scripts/time_advect.py C5 3 2>&1 | grep -v Warning
for f in paper_2004_02003_b200/var_*.so; do LAG_LIB=$f timeout 120 python scripts/time_advect.py C5 3; done 2>&1 | grep -v Warning
