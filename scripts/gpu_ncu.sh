#!/bin/bash
# GPU pass: build, GPU tests, bench, ncu full capture of the advect kernel, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-v1}
NCU=${2:-1}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?"
tail -c 2500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ "$NCU" = "1" ]; then
timeout 300 python scripts/profile_advect.py C5 20 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:advect -s 15 -c 1 \
    -o gpurun_out/prof_advect_$TAG python scripts/profile_advect.py C5 20 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full exit $?"; tail -2 gpurun_out/ncu_full_$TAG.log
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $BCMD > gpurun_out/bench_for_ncu.json 2>gpurun_out/bench_for_ncu.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches exit $?"
fi
