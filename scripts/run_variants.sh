cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 scripts/mgpu_check.py C1 0 2>&1 | grep -v "^\*\|OMP_NUM\|^$" | grep -v "^  File\|^    " | head -40
