# N=2: comm phases, bench (weak scaling C5), multi-GPU parity
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/comm_phases.py > gpurun_out/n2_phases.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err
