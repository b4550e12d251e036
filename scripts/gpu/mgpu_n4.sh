set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/n4_tests.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus 4 > gpurun_out/n4_bench.json 2> gpurun_out/n4_bench.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 \
    scripts/comm_phases.py > gpurun_out/n4_phases.log 2>&1
