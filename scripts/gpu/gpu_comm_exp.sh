cd "${GRAFT_REPO_ROOT:-/root/repo}"
for lib in liblag liblag_NOWAIT liblag_NOPULL liblag_NOPACK; do
  for fl in "" "--no-flush"; do
    LAG_LIB=paper_2004_02003_b200/$lib.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 scripts/comm_phases.py $fl > gpurun_out/ph_$lib$fl.txt 2>&1
    echo "== $lib $fl: $(python -c "
import json,sys
t=open('gpurun_out/ph_$lib$fl.txt').read(); d=json.loads(t[t.index('{'):])['max_over_ranks']
print({k:(round(v['pre_exchange_us'],1),round(v['advect_us'],1),round(v['us_per_cycle_event'],1)) for k,v in d.items()})")"
  done
done
