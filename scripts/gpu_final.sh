#!/bin/bash
# round evidence: build, GPU tests, smoke, bench N=1, launch list of the same bench, full ncu of advect
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r1}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench_$TAG.json
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $BCMD > gpurun_out/bench_for_ncu_$TAG.json 2>/dev/null && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches exit $?"
timeout 300 python scripts/profile_advect.py C5 20 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:advect -s 15 -c 1 \
    -o gpurun_out/prof_advect_$TAG python scripts/profile_advect.py C5 20 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full exit $?"
