cd "${GRAFT_REPO_ROOT:-/root/repo}"
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nproc
timeout 1500 python scripts/agreement.py C2 10 --save > gpurun_out/agree_C2.json 2> gpurun_out/agree_C2.err; echo "agree exit $?"
cp profiles/agreement_C2.json gpurun_out/ 2>/dev/null
tail -c 1500 gpurun_out/agree_C2.json; tail -3 gpurun_out/agree_C2.err
