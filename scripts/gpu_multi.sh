cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${1:-2}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
nvidia-smi -L
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 scripts/mgpu_check.py C2 33 > gpurun_out/mgpu_$N.log 2>&1; echo "mgpu exit $?"
grep '^{' gpurun_out/mgpu_$N.log; tail -20 gpurun_out/mgpu_$N.log | grep -v '^{' | tail -12
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench exit $?"
tail -c 2000 gpurun_out/bench_n$N.json; tail -5 gpurun_out/bench_n$N.err
