# A/B on one box: comm_phases and the bench's comm legs for two builds, interleaved
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
port=29580
for rep in 1 2; do
for v in ${VARIANTS:-liblag_prev liblag_new}; do
  port=$((port+1))
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port scripts/comm_phases.py > gpurun_out/ab_$v.json 2>/dev/null
  port=$((port+1))
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --no-secondary --no-e2e > gpurun_out/ab_bench_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
t = open(f"gpurun_out/ab_{v}.json").read(); d = json.loads(t[t.index("{"):])
p = d["max_over_ranks"]["comm_peer"]
t = open(f"gpurun_out/ab_bench_{v}.json").read(); b = json.loads(t[t.index("{"):].splitlines()[0])
c = b["comm"]["peer"]; o = b["comm"]["peer_overlap"]
print(f"{v:14s} phases: cycle {p['us_per_cycle_event']:.1f} pre {p['pre_exchange_us']:.1f} adv {p['advect_us']:.1f} | bench: bto {1e3*b['config']['ms_per_cycle']:.1f} peer {1e3*c['ms_per_cycle']:.1f} us/cycle ratio {c['bto_speedup']:.3f} | overlap {1e3*o['ms_per_cycle']:.1f} ratio {o['bto_speedup']:.3f}")
PY
done
done
