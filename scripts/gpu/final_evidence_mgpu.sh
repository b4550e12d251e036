# round-2 final multi-GPU evidence on a 4-GPU box: multi-GPU tests, bench at N=4 and N=2, comm phases at N=4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
set -x
mkdir -p gpurun_out/finm
timeout 1800 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/finm/tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
    bench.py --gpus 4 > gpurun_out/finm/bench_n4.json 2> gpurun_out/finm/bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
    bench.py --gpus 2 > gpurun_out/finm/bench_n2.json 2> gpurun_out/finm/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 \
    scripts/comm_phases.py > gpurun_out/finm/phases_n4.json 2> gpurun_out/finm/phases_n4.err
ls -la gpurun_out/finm
