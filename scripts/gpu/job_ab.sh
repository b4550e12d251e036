set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for lib in liblag_v3.so liblag.so; do
  LAG_LIB=paper_2004_02003_b200/$lib python scripts/time_advect.py C5 3
  LAG_LIB=paper_2004_02003_b200/$lib python scripts/time_advect.py C3 1
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
