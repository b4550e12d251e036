cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in liblag liblag_nopdl liblag liblag_nopdl; do
  LAG_LIB=$PWD/paper_2004_02003_b200/$v.so timeout 600 python scripts/tradeoff.py C4 2,2,2 --interval 100 --intervals 1 --delaunay-intervals 0 --tag tt_$v 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(1e3*d['bto_ms_per_cycle'],1), round(1e3*d['comm_ms_per_cycle'],1), round(d['bto_speedup_per_cycle_1gpu'],3))"
done
