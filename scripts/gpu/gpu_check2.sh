cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'ms/step', d['ms_per_step'], 'share', d['roofline']['kernel_share_of_step'], 'comm', d['comm']['value'])"
