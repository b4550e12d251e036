"""Summarise an ncu report: SOL, occupancy, stalls, per-opcode instruction mix.
usage: python scripts/ncu_summary.py gpurun_out/prof_X.ncu-rep [particles]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
parts = float(sys.argv[2]) if len(sys.argv) > 2 else None


def page(p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, vals = raw[0], raw[2]
R = dict(zip(hdr, vals))


def g(k):
    try:
        return float(R[k].replace(",", ""))
    except Exception:
        return float("nan")


keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    print(f"{k:70s} {R.get(k, '?')}")
tot = 0
rows = []
for h, v in zip(hdr, vals):
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h:
        x = float(v.replace(",", ""))
        rows.append((x, h))
        tot += x
print("stalls:")
for x, h in sorted(rows, reverse=True)[:8]:
    print(f"   {100 * x / tot:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = page("source")
sh, data = src[1], src[2:]
ix, ie, iw = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
T = S = 0
for r in data:
    try:
        n = float(r[ie] or 0)
        w = float(r[iw] or 0)
    except Exception:
        continue
    op = r[ix].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    o = o.split(".")[0]
    cnt[o] += n
    stall[o] += w
    T += n
    S += w
tiles = parts / 32 if parts else 1
print(f"warp-instructions per {'tile' if parts else 'launch'}: {T / tiles:.1f}")
print("  ".join(f"{o}:{n / tiles:.0f}({100 * stall[o] / max(S, 1):.0f}%)" for o, n in cnt.most_common(24)))
