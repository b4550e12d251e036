"""BTO speed-up paired with flow-map agreement on the SAME decomposition
(the paper's trade-off: speed-up P:511 vs accuracy Eq. 5/6).

For one configuration and block layout, on one GPU:
  * BTO: one context per block, one stream each (no communication);
  * COMM: the same blocks as one LAG_XCHG_LOCAL group (ghost copy + hand-off
    appends every cycle, return to origin at the write cycle), one stream
    per block;
  * per cycle the device time of the whole layout (the cycle of every block
    captured as a CUDA graph, fork to the blocks' streams and join back,
    replayed once between two events after an L2 flush) for both arms:
    BTO/COMM speed-up = mean COMM cycle time / mean BTO cycle time (write
    cycles excluded);
  * per interval: Eq. 5 over the seeds valid in the COMM map, with BTO holes
    reconstructed by Delaunay + barycentric interpolation (Qhull QJ
    over hole tiles, reading R12) on the host cores, and by GridFill
    (reading R18); Eq. 6 with C = cell side.
Writes profiles/tradeoff_<tag>.json.

  python scripts/tradeoff.py CONFIG LAYOUT [--intervals K] [--delaunay-intervals D]
         [--interval I] [--dtmul X] [--scale N] [--tag T]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("layout", help="blocks per axis, e.g. 2,1,1")
    ap.add_argument("--intervals", type=int, default=4)
    ap.add_argument("--delaunay-intervals", type=int, default=2)
    ap.add_argument("--interval", type=int, default=None)
    ap.add_argument("--dtmul", type=float, default=1.0, help="scale dt (CFL) by this factor")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--stride", type=int, default=None)
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    from oracle import metrics
    layout = tuple(int(x) for x in args.layout.split(","))
    nb = int(np.prod(layout))
    cfg = L.make_config(args.config, nranks=nb, scale=args.scale, interval=args.interval)
    cfg["layout"] = layout
    cfg["dt"] *= args.dtmul
    g = cfg["grid"]
    stride = args.stride or cfg["stride"]
    I = cfg["interval"]
    blocks = L.decompose(g, layout)
    main_s = torch.cuda.Stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def make(mode):
        ghost = 1 if mode == P.LAG_COMM else 0
        streams = [torch.cuda.Stream() for _ in blocks]
        cfgs = [P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=mode, ghost=ghost,
                              rank=b.rank if ghost else 0, nranks=nb if ghost else 1,
                              layout=layout if ghost else (1, 1, 1), stream=st.cuda_stream,
                              exchange=P.LAG_XCHG_LOCAL if ghost else 0) for b, st in zip(blocks, streams)]
        if ghost:
            grp = P.LocalGroup(cfgs)
            return dict(ctxs=grp.blocks, grp=grp, streams=streams, ghost=1)
        return dict(ctxs=[P.Context(c) for c in cfgs], grp=None, streams=streams, ghost=0)

    arms = {"bto": make(P.LAG_BTO), "comm": make(P.LAG_COMM)}
    for a in arms.values():
        a["n"] = [c.seed(stride) for c in a["ctxs"]]

    def window(arm, fn):
        """One cycle of every block, captured as a CUDA graph (fork from the
        capture stream to the blocks' streams, join back) and replayed once
        between two events: the device time of the layout's cycle without
        the host's launch overhead (eight blocks' calls would otherwise be
        host-bound)."""
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=main_s):
            ev = torch.cuda.Event()
            ev.record(main_s)
            for st in arm["streams"]:
                st.wait_event(ev)
            fn()
            for st in arm["streams"]:
                e = torch.cuda.Event()
                e.record(st)
                main_s.wait_event(e)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_s)
        gr.replay()
        e1.record(main_s)
        arm.setdefault("graphs", []).append(gr)      # alive until the events are read
        return e0, e1

    # global seed lattice (x fastest) and each block's seeds in it
    def lattice(lo, hi):
        ax = [np.arange(-(-lo[a] // stride) * stride, hi[a], stride) if a < g.dim else np.zeros(1, int)
              for a in range(3)]
        gz, gy, gx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1)
    gall = lattice((0, 0, 0), g.nodes)
    dims = [len(np.arange(0, g.nodes[a], stride)) if a < g.dim else 1 for a in range(3)]
    bidx = []
    for b in blocks:
        q = lattice(b.lo, b.hi) // stride
        bidx.append(q[:, 0] + dims[0] * (q[:, 1] + dims[1] * q[:, 2]))
    nall = gall.shape[0]
    start = np.stack([g.origin[a] + gall[:, a] * g.spacing[a] for a in range(g.dim)], 1)

    def cut(V, b, G):
        s_ = L.cut_block_slice(V, g, b, G).contiguous()
        if G:                    # ghost layers NaN: only the exchange may fill them
            for ax in range(g.dim):
                d = s_.dim() - 2 - ax
                s_.narrow(d, 0, 1).fill_(float("nan"))
                s_.narrow(d, s_.shape[d] - 1, 1).fill_(float("nan"))
        return s_

    cyc = {"bto": [], "comm": []}
    per = []
    t_cpu = 0.0
    prev = {"bto": None, "comm": None}       # this cycle's v_t = the previous call's v_t1 (in situ)
    for it in range(args.intervals):
        ev = {"bto": [], "comm": []}
        with torch.cuda.stream(main_s):
            for k in range(I):
                t = (it * I + k) * cfg["dt"]
                V0 = L.field_at_nodes(cfg["field"], g, t, device="cuda", backend="torch") if prev["bto"] is None else None
                V1 = L.field_at_nodes(cfg["field"], g, t + cfg["dt"], device="cuda", backend="torch")
                for name, arm in arms.items():
                    G = arm["ghost"]
                    sl = []
                    for i, b in enumerate(blocks):
                        s0 = prev[name][i] if prev[name] is not None else cut(V0, b, G)
                        sl.append((s0, cut(V1, b, G)))
                    prev[name] = [x[1] for x in sl]
                    torch.cuda.current_stream().synchronize()

                    def adv(arm=arm, sl=sl):
                        for c, (s0, s1) in zip(arm["ctxs"], sl):
                            c.advect(s0, s1, cfg["dt"])
                    ev[name].append(window(arm, adv))
            torch.cuda.synchronize()
        for name in ev:
            cyc[name] += [a.elapsed_time(b) for a, b in ev[name]]
        for arm in arms.values():
            arm["graphs"] = []
        # write cycle: both maps in global seed order
        maps = {}
        for name, arm in arms.items():
            end = np.zeros((nall, g.dim))
            st = np.zeros(nall, dtype=np.uint8)
            outs = [(torch.empty((n, g.dim), dtype=torch.float64, device="cuda"),
                     torch.empty((n,), dtype=torch.uint8, device="cuda")) for n in arm["n"]]
            for c, (e_, s_) in zip(arm["ctxs"], outs):
                c.extract(end=e_, status=s_)
            torch.cuda.synchronize()
            for (e_, s_), ix in zip(outs, bidx):
                end[ix] = e_.cpu().numpy()
                st[ix] = s_.cpu().numpy()
            maps[name] = (end, st)
        t1 = time.time()
        row = {"interval": it}
        for method in (["delaunay"] if it < args.delaunay_intervals else []) + ["gridfill"]:
            r = metrics.agreement(g, gall, start, maps["bto"][0], maps["bto"][1], maps["comm"][0],
                                  maps["comm"][1], stride, method=method)
            row[method] = {k: r[k] for k in ("L", "max_l2", "accuracy", "holes", "excluded", "compared")}
            row["discarded_pct"] = 100.0 * r["discarded"] / r["seeded"]
            row["comm_exits_pct"] = 100.0 * float((maps["comm"][1] != 0).mean())
        t_cpu += time.time() - t1
        per.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    for arm in arms.values():
        if arm["grp"] is not None:
            arm["grp"].close()
        else:
            for c in arm["ctxs"]:
                c.close()
    C = metrics.cell_side(g)
    out = {"config": cfg["name"], "layout": list(layout), "grid": list(g.nodes), "stride": stride,
           "interval": I, "intervals": args.intervals, "dt": cfg["dt"], "dtmul": args.dtmul,
           "seeds": int(nall), "cell_side_C": C,
           "bto_ms_per_cycle": float(np.mean(cyc["bto"])), "comm_ms_per_cycle": float(np.mean(cyc["comm"])),
           "bto_speedup_per_cycle_1gpu": float(np.mean(cyc["comm"]) / np.mean(cyc["bto"])),
           "discarded_pct": float(np.mean([r["discarded_pct"] for r in per])),
           "cpu_seconds_metric": t_cpu, "cpu_cores": os.cpu_count(),
           "per_interval": per}
    for method in ("delaunay", "gridfill"):
        rows = [r[method] for r in per if method in r]
        if rows:
            Lm = float(np.mean([r["L"] for r in rows]))
            gmax, amax = metrics.max_l2_stats([r["max_l2"] for r in rows])
            out[method] = {"intervals": len(rows), "total_average_L2": Lm,
                           "accuracy_pct": float(np.mean([r["accuracy"] for r in rows])),
                           "accuracy_pct_paper_style": metrics.paper_printed_accuracy(Lm, C),
                           "greatest_max_L2": gmax, "average_max_L2": amax,
                           "excluded_outside_hull": int(sum(r["excluded"] for r in rows))}
    out["method"] = ("one GPU; BTO = one context per block, COMM = LAG_XCHG_LOCAL group of the same "
                     "blocks; per-cycle device time of the whole layout (each cycle captured as a CUDA graph "
                     "and replayed once, L2 flushed before each cycle); "
                     "Eq. 5/6 over seeds valid in COMM, holes by Delaunay+barycentric (Qhull QJ, first "
                     f"{args.delaunay_intervals} intervals) and GridFill (all intervals)")
    print(json.dumps({k: v for k, v in out.items() if k != "per_interval"}), flush=True)
    tag = args.tag or f"{cfg['name']}_{'x'.join(map(str, layout))}_i{I}" + (f"_dt{args.dtmul:g}" if args.dtmul != 1 else "")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"tradeoff_{tag}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
