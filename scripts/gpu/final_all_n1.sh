# final round-2 evidence at N=1 (the driver's round-end sequence): GPU tests, smoke, bench, reference arm
set -x
timeout 1000 python -m pytest tests -m gpu -q > gpurun_out/z_tests.log 2>&1
python __graft_entry__.py smoke > gpurun_out/z_smoke.log 2>&1
python bench.py > gpurun_out/z_bench_n1.json 2> gpurun_out/z_bench_n1.err
python bench.py --impl reference > gpurun_out/z_ref.json 2> gpurun_out/z_ref.err
