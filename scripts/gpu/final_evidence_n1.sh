# round-2 final evidence at N=1: GPU tests, smoke, bench, reference arm, launch list, full ncu (C5 cycle 12, C3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
set -x
mkdir -p gpurun_out/fin
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin/tests_n1.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log
timeout 900 python bench.py > gpurun_out/fin/bench_n1.json 2> gpurun_out/fin/bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/fin/ref.json 2> gpurun_out/fin/ref.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary"
timeout 300 $BCMD > gpurun_out/fin/bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"advect|seed_kernel|extract|append|halo|local_|route|peer" -c 3000 --csv \
      --log-file gpurun_out/fin/launches.csv $BCMD > gpurun_out/fin/ncu_launch.log 2>&1
timeout 300 python scripts/time_advect.py C5 1 > gpurun_out/fin/plain_c5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 37 -c 1 \
      -o gpurun_out/fin/prof_c5 python scripts/time_advect.py C5 1 > gpurun_out/fin/ncu_c5.log 2>&1
timeout 300 python scripts/time_advect.py C3 0 > gpurun_out/fin/plain_c3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 16 -c 1 \
      -o gpurun_out/fin/prof_c3 python scripts/time_advect.py C3 0 > gpurun_out/fin/ncu_c3.log 2>&1
ls -la gpurun_out/fin
