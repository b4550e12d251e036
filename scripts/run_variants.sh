cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29558 bench.py --gpus $N --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_peer_n$N.json 2> gpurun_out/bench_peer_n$N.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_peer_n$N.json'))
print('BTO', d['value'], 'ms/cyc', d['config']['ms_per_cycle'])
for k in ('nccl','peer'):
    if k in d['comm']: print(k, d['comm'][k])
print('secondary', d['secondary']['value'], d['secondary']['roofline']['frac'])"
