# N = 1, 2, 4 back to back on one 4-GPU box (the driver's scaling sequence), BTO headline + comm legs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/scale
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/scale/n1.json 2> gpurun_out/scale/n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 > gpurun_out/scale/n2.json 2> gpurun_out/scale/n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 > gpurun_out/scale/n4.json 2> gpurun_out/scale/n4.err
python - <<'PY'
import json
rows = {}
for n in (1, 2, 4):
    t = open(f"gpurun_out/scale/n{n}.json").read()
    d = json.loads(t[t.index("{"):].strip().splitlines()[-1])
    rows[n] = {"value": d["value"], "ms_per_cycle": d["config"]["ms_per_cycle"], "comm_value": d["comm"]["value"],
               "bto_speedup": d["comm"]["bto_speedup"], "e2e": d["e2e"]["value"], "clocks": d["clocks"]}
for n in (2, 4):
    rows[n]["weak_scaling_efficiency"] = rows[n]["value"] / (n * rows[1]["value"])
json.dump({"box": "one 4-GPU B200 box, N = 1, 2, 4 back to back (bench.py, C5 weak scaling)", "rows": rows},
          open("gpurun_out/scale/scale_n124.json", "w"), indent=1)
print(json.dumps({n: {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k != "clocks"} for n, r in rows.items()}))
PY
