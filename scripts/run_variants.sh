cd "${GRAFT_REPO_ROOT:-/root/repo}"
for f in paper_2004_02003_b200/var_*.so; do LAG_LIB=$f timeout 120 python scripts/time_advect.py C5 3; done 2>&1 | grep -v Warning
