cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/tl_flush gpurun_out/tl_noflush
LAG_TL_DIR=gpurun_out/tl_flush LAG_LIB=paper_2004_02003_b200/liblag_TL.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-2} --master-addr 127.0.0.1 --master-port 29559 scripts/comm_phases.py > gpurun_out/tl_flush/out.txt 2>&1
LAG_TL_DIR=gpurun_out/tl_noflush LAG_LIB=paper_2004_02003_b200/liblag_TL.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-2} --master-addr 127.0.0.1 --master-port 29559 scripts/comm_phases.py --no-flush > gpurun_out/tl_noflush/out.txt 2>&1
ls gpurun_out/tl_flush gpurun_out/tl_noflush
