cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LAG_LIB=$PWD/paper_2004_02003_b200/liblag_TL.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 scripts/gpu/tl_peer.py > gpurun_out/tl_peer.log 2>&1
tail -20 gpurun_out/tl_peer.log
