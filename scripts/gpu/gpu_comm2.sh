cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 scripts/comm_phases.py > gpurun_out/phases2.txt 2>&1; echo "phases exit $?"
grep -A30 max_over gpurun_out/phases2.txt | head -30
