cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pt4.log 2>&1; echo "pytest exit $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pt4.log | head -10
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 scripts/comm_phases.py > gpurun_out/ph4.log 2>&1; echo "phases exit $?"
python - <<'PY'
import json
t=open('gpurun_out/ph4.log').read(); j=t[t.index('{'):t.rindex('}')+1]; d=json.loads(j)
for k,v in d['max_over_ranks'].items(): print(k, {kk: round(vv,1) for kk,vv in v.items()})
PY
