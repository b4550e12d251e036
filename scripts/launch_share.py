"""Summarise an ncu launch list (gpu__time_duration.sum per launch): per
kernel-name totals and the advect kernel's share of the library's kernels.
usage: python scripts/launch_share.py gpurun_out/launches_X.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ik]
    short = name.split("(")[0].replace("void ", "")[:60]
    tot[short][0] += 1
    tot[short][1] += float(r[iv].replace(",", ""))
lag = {k: v for k, v in tot.items() if k.startswith("lag::")}
lag_ns = sum(v[1] for v in lag.values())
print(f"{'kernel':62s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share of lag':>12s}")
for k, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    share = f"{100 * ns / lag_ns:6.1f}%" if k in lag else ""
    print(f"{k:62s} {n:8d} {ns / 1e3:10.1f} {ns / n / 1e3:9.2f} {share:>12s}")
