cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LAG_LIB=$PWD/paper_2004_02003_b200/liblag_TL.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 scripts/gpu/tl_peer.py > gpurun_out/tl_peer_new.log 2>&1
mv gpurun_out/tl_peer_n2.json gpurun_out/tl_peer_n2_new.json
grep us/cycle gpurun_out/tl_peer_new.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 scripts/comm_phases.py > gpurun_out/phases_new.json 2>gpurun_out/phases_new.err
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_new.log 2>&1; tail -3 gpurun_out/multi_new.log
