cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in ${VARIANTS:-liblag_TL2}; do
echo "== $v"
LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 scripts/gpu/tl_overlap.py 2>&1 | grep -v "^\*\|OMP\|NCCL version"
done
