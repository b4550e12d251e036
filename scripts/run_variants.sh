cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python scripts/time_advect.py C5 3 2>&1 | grep -v Warning
timeout 120 python scripts/time_advect.py C5 3 --warm 2>&1 | grep -v Warning
timeout 120 python scripts/time_advect.py C3 2 2>&1 | grep -v Warning
timeout 120 python scripts/time_advect.py C3 2 --warm 2>&1 | grep -v Warning
