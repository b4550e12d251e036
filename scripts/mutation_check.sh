#!/bin/bash
# Mutation check of the oracle's pins: each line plants one plausible mistake
# in a scratch copy of oracle/ and runs tests/test_oracle_pins.py there; every
# mutation must make at least one pin fail ("N failed").
# Two mutants are left out on purpose because they are equivalent on every
# input the method sees: C = J^T J -> J J^T in ftle.py (same nonzero
# eigenvalues, so the same lambda_max) and min -> max over axes in
# metrics.cell_side (every grid the paper prints an accuracy for is
# isotropic; reading R10).
# usage: bash scripts/mutation_check.sh   (from the repo root, CPU only)
cd "$(dirname "$0")/.."
run() {  # name file old new
  d=$(mktemp -d); cp -r oracle lag_inputs tests $d/; rm -f $d/oracle/liboracle.so
  python3 - "$d/oracle/$2" "$3" "$4" <<'PY'
import sys
p,old,new=sys.argv[1:4]
s=open(p).read(); assert old in s, old; open(p,'w').write(s.replace(old,new,1))
PY
  r=$(cd $d && timeout 600 python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider 2>&1 | tail -1)
  echo "$1: $r"
}
run face0 lag_oracle.c "    double best = INFINITY;" "    return 0.0; double best = INFINITY;"
run touchshift lag_oracle.c "for (int a = 0; a < g->dim; ++a) n[a] = i[a] + ((corner >> a) & 1);" "for (int a = 0; a < g->dim; ++a) n[a] = i[a] + ((corner >> a) & 1) + (a == 0);"
run longest metrics.py "best = spans.min(axis=1)" "best = np.where(spans < np.iinfo(np.int64).max, spans, -1).max(axis=1)"
run margin0 metrics.py "margin: int = 3" "margin: int = 0"
run alpha lag_oracle.c "RK_ALPHA[4] = {0.0, 0.5, 0.5, 1.0}" "RK_ALPHA[4] = {0.0, 0.5, 0.5, 0.5}"
run beta lag_oracle.c "RK_BETA[4]  = {0.0, 0.5, 0.5, 1.0}" "RK_BETA[4]  = {0.0, 0.5, 1.0, 1.0}"
run bweights lag_oracle.c "RK_B[4]     = {1.0, 2.0, 2.0, 1.0}" "RK_B[4]     = {1.0, 2.0, 1.0, 2.0}"
run sixth lag_oracle.c "xn[a] = x[a] + dt / 6.0 * sum;" "xn[a] = x[a] + dt / 5.0 * sum;"
run closedhi lag_oracle.c "if (!(q[a] < hi_x)) return 0;" "if (!(q[a] <= hi_x)) return 0;"
run noupdatetest lag_oracle.c "        int outcome = classify(g, lo, hi, mode, xn);" "        int outcome = ORC_VALID; (void)xn;"
run interpw lag_oracle.c "w *= delta ? f[a] : (1.0 - f[a]);" "w *= delta ? (1.0 - f[a]) : f[a];"
run seedexcl lag_oracle.c "if (mind && s > 0) {" "if (mind) {"
run eq5div metrics.py "sum()) / p" "sum()) / (p + 1)"
run eq5sq metrics.py "np.sqrt(((b - m) ** 2).sum(axis=1)).sum()" "((b - m) ** 2).sum(axis=1).sum()"
run eq6 metrics.py "return (C - L) / C * 100.0" "return (C - L) / L * 100.0"
run maxavg metrics.py "return max(vals), sum(vals) / len(vals)" "return max(vals), max(vals)"
run ftlelog ftle.py "np.log(np.sqrt(lam[ok]))" "np.log(lam[ok])"
run ftlemin ftle.py "np.linalg.eigvalsh(C[fin])[:, -1]" "np.linalg.eigvalsh(C[fin])[:, 0]"
run ftleT ftle.py "/ abs(T)" "/ T"
run ftleedge ftle.py "axis=npax, edge_order=1" "axis=npax, edge_order=2"
run kuhnw0 pathline.py "w[:, 0] = 1.0 - fs[:, 0]" "w[:, 0] = fs[:, 0]"
run kuhnord pathline.py 'np.argsort(-f, axis=1, kind="stable")' 'np.argsort(f, axis=1, kind="stable")'
run stitchcube pathline.py "i = np.minimum(np.floor(uu).astype(np.int64), dims - 2)" "i = np.floor(uu).astype(np.int64)"
