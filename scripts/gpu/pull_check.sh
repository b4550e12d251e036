cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pull_multi.log 2>&1; tail -3 gpurun_out/pull_multi.log
VARIANTS=liblag bash scripts/gpu/phases_variants.sh
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multi.py > gpurun_out/pull_gpu.log 2>&1; tail -3 gpurun_out/pull_gpu.log
