cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 scripts/mgpu_check.py C2 33 > gpurun_out/mg.log 2>&1; echo "mgpu exit $?"
grep -E "^\{" gpurun_out/mg.log | cut -c1-260
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29559 scripts/comm_phases.py > gpurun_out/ph.log 2>&1; echo "phases exit $?"
python - <<'PY'
import json,re
t=open('gpurun_out/ph.log').read(); j=t[t.index('{'):t.rindex('}')+1]; d=json.loads(j)
for k,v in d['max_over_ranks'].items(): print(k, {kk: round(vv,1) for kk,vv in v.items()})
PY
