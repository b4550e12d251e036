bash scripts/gpu/job_variants.sh liblag.so liblag_cs.so liblag_na.so liblag_el.so > gpurun_out/hints.log 2>&1
LAG_LIB=paper_2004_02003_b200/liblag_noload.so python scripts/time_advect.py C5 1 > gpurun_out/nl_plain.log 2>&1 && \
LAG_LIB=paper_2004_02003_b200/liblag_noload.so ncu --set full --clock-control none --import-source on -k regex:advect_kernel -s 37 -c 1 \
    -o gpurun_out/prof_noload python scripts/time_advect.py C5 1 > gpurun_out/nl_ncu.log 2>&1
