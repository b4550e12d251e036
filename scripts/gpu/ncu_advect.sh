# full ncu capture of one advect launch (cycle 12 of the second C5 interval)
python scripts/time_advect.py C5 1 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 37 -c 1 \
    -o gpurun_out/prof_c5 python scripts/time_advect.py C5 1 > gpurun_out/ncu.log 2>&1
