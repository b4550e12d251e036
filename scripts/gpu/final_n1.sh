# round-2 evidence at N=1: bench (default), launch list of our kernels, full ncu of advect on C3, smoke
set -x
python __graft_entry__.py smoke > gpurun_out/f_smoke.log 2>&1
python bench.py > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary"
timeout 300 $BCMD > gpurun_out/f_bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"advect|seed_kernel|extract|append|halo|local_|route" -c 3000 --csv \
      --log-file gpurun_out/f_launches.csv $BCMD > gpurun_out/f_ncu_launch.log 2>&1
python scripts/time_advect.py C3 0 > gpurun_out/f_plain_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 16 -c 1 \
      -o gpurun_out/f_prof_c3 python scripts/time_advect.py C3 0 > gpurun_out/f_ncu_c3.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
