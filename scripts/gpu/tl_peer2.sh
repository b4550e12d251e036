cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in TL TLf; do
LAG_LIB=$PWD/paper_2004_02003_b200/liblag_$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 scripts/gpu/tl_peer.py > gpurun_out/tl_peer_$v.log 2>&1
mv gpurun_out/tl_peer_n2.json gpurun_out/tl_peer_n2_$v.json
grep us/cycle gpurun_out/tl_peer_$v.log
done
