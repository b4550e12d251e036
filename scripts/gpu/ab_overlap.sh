# A/B of two builds on one 2-GPU box: comm phases (overlap transport) + the multi-GPU tests on the new build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
port=29590
for rep in 1 2; do
for v in ${VARIANTS:-liblag_prev liblag_new}; do
  port=$((port+1))
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port scripts/comm_phases.py > gpurun_out/abo_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
t = open(f"gpurun_out/abo_{v}.json").read(); d = json.loads(t[t.index("{"):])
m = d["max_over_ranks"]
print(v, {k: round(m[k]["us_per_cycle_event"], 1) for k in m}, {k: round(x, 1) for k, x in m["comm_peer_overlap"].items()})
PY
done
done
[ -n "$TESTS" ] && timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
