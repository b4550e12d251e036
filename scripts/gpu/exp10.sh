cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build >/dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 scripts/mgpu_check.py C2 33 2>&1 | grep '^{' | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 scripts/comm_phases.py 2>&1 | grep -A6 '"comm_peer'
