cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
L=paper_2004_02003_b200
for o in 4 3 2 1; do echo "== base occ $o"; LAG_ADV_OCC=$o LAG_LIB=$L/liblag.so timeout 300 python scripts/time_advect.py C5 2 2>&1 | tail -1; done
for o in 4 2; do echo "== nl occ $o"; LAG_ADV_OCC=$o LAG_LIB=$L/liblag_nl.so timeout 300 python scripts/time_advect.py C5 2 2>&1 | tail -1; done
for v in nl6 m6; do echo "== $v"; LAG_LIB=$L/liblag_$v.so timeout 300 python scripts/time_advect.py C5 2 2>&1 | tail -1; done
