# round evidence: GPU tests, advect timing, launch list and full ncu of the advect kernel (C5 cycle 12, C3)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_tests.log 2>&1
python scripts/time_advect.py C5 3 > gpurun_out/ev_time.log 2>&1
python scripts/time_advect.py C3 1 >> gpurun_out/ev_time.log 2>&1
python scripts/gpu/pitch_probe.py > gpurun_out/ev_pitch.log 2>&1
python bench.py --steps 2 --warmup 1 --no-comm --no-e2e --no-cpu --no-secondary > gpurun_out/ev_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-comm --no-e2e --no-cpu --no-secondary > gpurun_out/ev_ncu_launch.log 2>&1
python scripts/time_advect.py C5 1 > gpurun_out/ev_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 37 -c 1 \
    -o gpurun_out/ev_prof_c5 python scripts/time_advect.py C5 1 > gpurun_out/ev_ncu_c5.log 2>&1
python scripts/time_advect.py C3 0 > gpurun_out/ev_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 16 -c 1 \
    -o gpurun_out/ev_prof_c3 python scripts/time_advect.py C3 0 > gpurun_out/ev_ncu_c3.log 2>&1
ls -la gpurun_out
