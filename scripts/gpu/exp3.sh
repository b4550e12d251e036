cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
L=paper_2004_02003_b200
for args in "C5 3" "C5 3 --warm" "C5 3 --frozen" "C5 3 --warm --frozen"; do
  echo "== rel $args"; LAG_LIB=$L/liblag_rel.so timeout 300 python scripts/time_advect.py $args 2>&1 | tail -1
done
echo "== nl"; LAG_LIB=$L/liblag_nl.so timeout 300 python scripts/time_advect.py C5 3 2>&1 | tail -1
