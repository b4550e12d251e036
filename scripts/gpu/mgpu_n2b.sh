set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/n2b_tests.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/comm_phases.py > gpurun_out/n2b_phases.log 2>&1
