cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err
echo "rc=$?"
python - <<'PY'
import json
t = open("gpurun_out/n2_bench.json").read()
d = json.loads(t[t.index("{"):].splitlines()[0]) if "{" in t else {}
c = d.get("comm", {})
print("value", d.get("value"), "ms/cycle", d.get("config", {}).get("ms_per_cycle"))
for k, v in c.items():
    if isinstance(v, dict): print(k, {a: b for a, b in v.items() if a in ("value", "ms_per_cycle", "bto_speedup")})
PY
