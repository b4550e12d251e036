set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/y_tests.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 4 > gpurun_out/y_bench_n4.json 2> gpurun_out/y_bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
    bench.py --gpus 2 > gpurun_out/y_bench_n2.json 2> gpurun_out/y_bench_n2.err
