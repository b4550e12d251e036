# A/B of two builds on one GPU: GPU tests on the new build, then the bench (C5 headline only) for each, twice
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2; }
for rep in 1 2; do
for v in ${VARIANTS:-liblag_prev liblag_new}; do
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 600 python bench.py --no-cpu --no-e2e --no-secondary --no-comm > gpurun_out/abn1_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/abn1_{v}.json").read().strip().splitlines()[-1])
print(f"{v:14s} value {d['value']/1e9:.3f} G  ms/step {d['ms_per_step']:.4f}  us/cycle {1e3*d['config']['ms_per_cycle']:.2f}")
PY
done
done
