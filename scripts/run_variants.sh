cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
timeout 120 python scripts/time_advect.py C5 3 2>&1 | grep -v Warning
timeout 120 python scripts/time_advect.py C5 3 --frozen 2>&1 | grep -v Warning
timeout 120 python scripts/time_advect.py C3 2 --frozen 2>&1 | grep -v Warning
