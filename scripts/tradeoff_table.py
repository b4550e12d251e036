"""Collect scripts/tradeoff.py results (profiles/tradeoff_*.json) into one
table: per configuration and decomposition, the BTO-over-COMM per-cycle
speed-up on one GPU next to the flow-map agreement (Eq. 5/6) of the same run,
and the multi-GPU speed-ups of bench.py where they exist.

  python scripts/tradeoff_table.py [files...]   -> profiles/tradeoff_table.json + markdown on stdout
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    files = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "profiles", "tradeoff_*.json")))
    # the flow maps are deterministic (bitwise), so a timing refresh (file
    # ending in _t.json) keeps the agreement columns of the full run of the
    # same row and replaces only its per-cycle times
    full = {}
    for f in files:
        if f.endswith("tradeoff_table.json") or f.endswith("_t.json"):
            continue
        d = json.load(open(f))
        full[(d["config"], tuple(d["layout"]), d["interval"], d.get("dtmul", 1.0))] = d
    merged = []
    for f in files:
        if f.endswith("tradeoff_table.json"):
            continue
        d = json.load(open(f))
        key = (d["config"], tuple(d["layout"]), d["interval"], d.get("dtmul", 1.0))
        if f.endswith("_t.json"):
            base = full.get(key)
            if base:                       # agreement of the full run (more intervals), timing of the refresh
                for m in ("delaunay", "gridfill"):
                    if m in base:
                        d[m] = base[m]
                d["discarded_pct"] = base["discarded_pct"]
                d["intervals"] = base["intervals"]
            d["_timing_from"] = os.path.relpath(f, ROOT)
            merged.append((f, d))
        elif not os.path.exists(f[:-5] + "_t.json"):
            merged.append((f, d))
    rows = []
    for f, d in merged:
        row = {"config": d["config"], "layout": "x".join(map(str, d["layout"])), "stride": d["stride"],
               "interval": d["interval"], "dtmul": d.get("dtmul", 1.0), "intervals": d["intervals"],
               "seeds": d["seeds"], "bto_us_per_cycle": 1e3 * d["bto_ms_per_cycle"],
               "comm_us_per_cycle": 1e3 * d["comm_ms_per_cycle"],
               "bto_speedup_per_cycle_1gpu": d["bto_speedup_per_cycle_1gpu"],
               "discarded_pct": d["discarded_pct"], "file": os.path.relpath(f, ROOT)}
        for m in ("delaunay", "gridfill"):
            if m in d:
                row[f"{m}_accuracy_pct"] = d[m]["accuracy_pct"]
                row[f"{m}_L"] = d[m]["total_average_L2"]
                row[f"{m}_max_L2"] = d[m]["greatest_max_L2"]
                row[f"{m}_intervals"] = d[m]["intervals"]
                row[f"{m}_excluded"] = d[m]["excluded_outside_hull"]
        rows.append(row)
    json.dump({"rows": rows, "source": "scripts/tradeoff.py (one GPU: BTO contexts vs a LAG_XCHG_LOCAL COMM "
                                       "group of the same blocks; Eq. 5/6 over seeds valid in COMM)"},
              open(os.path.join(ROOT, "profiles", "tradeoff_table.json"), "w"), indent=1)
    print("| Config | Layout | Stride | Interval | dt x | BTO µs/cycle | COMM µs/cycle | BTO/COMM | "
          "Discarded % | Accuracy % Delaunay (intervals) | Accuracy % GridFill (intervals) | Max L2 (Delaunay) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        dl = (f"{r['delaunay_accuracy_pct']:.3f} ({r['delaunay_intervals']})" if "delaunay_accuracy_pct" in r else "—")
        gf = (f"{r['gridfill_accuracy_pct']:.3f} ({r['gridfill_intervals']})" if "gridfill_accuracy_pct" in r else "—")
        mx = f"{r['delaunay_max_L2']:.2e}" if "delaunay_max_L2" in r else "—"
        print(f"| {r['config']} | {r['layout']} | {r['stride']} | {r['interval']} | {r['dtmul']:g} | "
              f"{r['bto_us_per_cycle']:.1f} | {r['comm_us_per_cycle']:.1f} | {r['bto_speedup_per_cycle_1gpu']:.2f} | "
              f"{r['discarded_pct']:.2f} | {dl} | {gf} | {mx} |")


if __name__ == "__main__":
    main()
