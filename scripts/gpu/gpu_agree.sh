cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() { timeout 1500 python scripts/agreement.py "$@" --save > /dev/null 2> gpurun_out/agree_err_$1_$2.log; echo "agree $* exit $?"; }
run C2 10 --recon gridfill
run C4 4 --interval 10 --recon gridfill
run C4 2 --interval 50 --recon gridfill
run C4 2 --interval 100 --recon gridfill
run C3 4 --recon gridfill --layout 2,2,2
run C2 4 --interval 50 --recon gridfill
run C2 2 --interval 100 --recon gridfill
cp profiles/agreement_*.json gpurun_out/
for f in profiles/agreement_*gridfill.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['config'], d['interval'], 'acc', round(d['accuracy_pct'],4), 'L', d['total_average_L2'], 'disc%', round(d['discarded_pct'],2), 'gmax', d['greatest_max_L2'], 'amax', d['average_max_L2'], 'excl', d['excluded_outside_hull'], 'cpu_s', round(d['cpu_seconds'],1))"; done
