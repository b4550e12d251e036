cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=.
python __graft_entry__.py build >/dev/null 2>&1
for s in 0 12; do
timeout 600 ncu --set full --clock-control none -k regex:advect -s $s -c 1 -f -o gpurun_out/prof_cyc$s python scripts/profile_advect.py C5 20 > gpurun_out/ncu_cyc$s.log 2>&1; echo "ncu $s exit $?"
done
