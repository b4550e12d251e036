# time advect variants: bash scripts/gpu/job_variants.sh lib1.so lib2.so ...
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for lib in "$@"; do
  LAG_LIB=paper_2004_02003_b200/$lib python scripts/time_advect.py C5 3
  LAG_LIB=paper_2004_02003_b200/$lib python scripts/time_advect.py C3 1
done
