cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
port=29570
for v in ${VARIANTS:-liblag}; do
  port=$((port+1))
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port scripts/comm_phases.py > gpurun_out/phases_$v.json 2> gpurun_out/phases_$v.err
  echo "$v rc=$?"
  python - "$v" <<'PY'
import json, sys
try:
    t = open(f"gpurun_out/phases_{sys.argv[1]}.json").read()
    d = json.loads(t[t.index("{"):])
    for k, v in d["max_over_ranks"].items(): print(" ", k, {a: round(b, 1) for a, b in v.items()})
except Exception as e:
    print("no json", e)
PY
done
