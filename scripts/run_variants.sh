cd "${GRAFT_REPO_ROOT:-/root/repo}"
export LAG_LIB=
timeout 120 python scripts/profile_advect.py C5 20 > gpurun_out/plain_v4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advect -s 15 -c 1 -o gpurun_out/prof_advect_v4 python scripts/profile_advect.py C5 20 > gpurun_out/ncu_v4.log 2>&1; echo ncu $?
