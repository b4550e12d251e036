# N=1: GPU tests, the advect timing per cycle position, and the bench (first-cycle frame change)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c0_tests.log 2>&1; tail -2 gpurun_out/c0_tests.log
timeout 300 python scripts/time_advect.py C5 1 2>&1 | tail -2
timeout 300 python scripts/time_advect.py C4 0 2>&1 | tail -2
timeout 300 python scripts/time_advect.py C3 0 2>&1 | tail -2
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/c0_bench.json 2> gpurun_out/c0_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c0_bench.json").read().strip().splitlines()[-1])
print("C5", d["value"] / 1e9, 1e3 * d["config"]["ms_per_cycle"], d["roofline"]["frac"])
print("C4", {k: (round(v["value"] / 1e9, 2), round(v["roofline"]["frac"], 3)) for k, v in d["c4"].items() if k.startswith("interval")})
print("C3", d["secondary"]["value"] / 1e9, d["secondary"]["roofline"]["frac"], "C2", d["c2"]["bto"]["value"] / 1e9, d["c2"]["comm"]["value"] / 1e9)
PY
