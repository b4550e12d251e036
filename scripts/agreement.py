"""BTO-vs-COMM flow-map agreement (the paper's accuracy metric).

Runs the product path on the GPU for `intervals` intervals of a config:
  * BTO: one context per block of the layout (all on this GPU);
  * COMM flow map: one context over the whole domain (R = 1, which equals the
    decomposed COMM run bitwise — scripts/mgpu_check.py — P:612-614);
then on the host CPU (oracle/metrics.py, test/measurement infrastructure):
  per interval, over seeds valid in COMM: b = BTO end, or for BTO holes its
  Delaunay-barycentric reconstruction from the valid basis flows around it
  (P:262-274); L = Eq. 5; accuracy = Eq. 6 with C = cell side.
Prints one JSON line (and writes it to profiles/agreement_<config>.json with --save).

  python scripts/agreement.py [config] [intervals] [--scale N] [--stride S] [--interval I] [--save]
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


def ctx_for(cfg, block, stream):
    g = cfg["grid"]
    return P.Context(P.make_config(g.dim, g.nodes, g.origin, g.spacing, block.lo, block.hi,
                                   stream=stream.cuda_stream))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("intervals", nargs="?", type=int, default=10)
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--stride", type=int, default=None)
    ap.add_argument("--interval", type=int, default=None)
    ap.add_argument("--save", action="store_true")
    ap.add_argument("--recon", default="delaunay", choices=["delaunay", "gridfill", "gpu-gridfill"],
                    help="gpu-gridfill: holes filled by lag_gridfill (CUDA), cross-checked bitwise "
                         "against the oracle's GridFill on the first interval")
    ap.add_argument("--tag", default="")
    ap.add_argument("--layout", default=None, help="blocks per axis, e.g. 2,2,2 (default: the config's)")
    args = ap.parse_args()
    from oracle import metrics
    cfg = L.make_config(args.config, scale=args.scale, interval=args.interval)
    g = cfg["grid"]
    stride = args.stride or cfg["stride"]
    I = cfg["interval"]
    if args.layout:
        cfg["layout"] = tuple(int(x) for x in args.layout.split(","))
    blocks = L.decompose(g, cfg["layout"])
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    s = torch.cuda.current_stream()
    ctxs = [ctx_for(cfg, b, s) for b in blocks]
    cw = ctx_for(cfg, whole, s)
    ns = [c.seed(stride) for c in ctxs]
    nw = cw.seed(stride)
    # global seed order of each block's seeds (x fastest), for assembling the BTO map
    def lattice(lo, hi):
        ax = [np.arange(-(-lo[a] // stride) * stride, hi[a], stride) if a < g.dim else np.zeros(1, int)
              for a in range(3)]
        gz, gy, gx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1)
    gall = lattice((0, 0, 0), g.nodes)
    dims = [len(np.arange(0, g.nodes[a], stride)) if a < g.dim else 1 for a in range(3)]
    def gidx(gg):
        q = gg // stride
        return q[:, 0] + dims[0] * (q[:, 1] + dims[1] * q[:, 2])
    bidx = [gidx(lattice(b.lo, b.hi)) for b in blocks]
    per, t_gpu, t_cpu, t_fill = [], 0.0, 0.0, 0.0
    for it in range(args.intervals):
        t0 = time.time()
        ext = [L.block_slice_extent(g, b, 0) for b in blocks]
        for k in range(I):
            t = (it * I + k) * cfg["dt"]
            V0 = L.field_at_nodes(cfg["field"], g, t, device="cuda", backend="torch")
            V1 = L.field_at_nodes(cfg["field"], g, t + cfg["dt"], device="cuda", backend="torch")
            cw.advect(V0.contiguous(), V1.contiguous(), cfg["dt"])
            for c, b, e in zip(ctxs, blocks, ext):
                sl0 = V0[b.lo[2]:b.lo[2] + e[2], b.lo[1]:b.lo[1] + e[1], b.lo[0]:b.lo[0] + e[0]].contiguous()
                sl1 = V1[b.lo[2]:b.lo[2] + e[2], b.lo[1]:b.lo[1] + e[1], b.lo[0]:b.lo[0] + e[0]].contiguous()
                c.advect(sl0, sl1, cfg["dt"])
        start = torch.empty((nw, g.dim), dtype=torch.float64, device="cuda")
        m_end = torch.empty_like(start)
        m_st = torch.empty((nw,), dtype=torch.uint8, device="cuda")
        cw.extract(start, m_end, m_st)
        b_end = np.zeros((nw, g.dim))
        b_st = np.zeros(nw, dtype=np.uint8)
        for c, n, ix in zip(ctxs, ns, bidx):
            e_ = torch.empty((n, g.dim), dtype=torch.float64, device="cuda")
            s_ = torch.empty((n,), dtype=torch.uint8, device="cuda")
            c.extract(end=e_, status=s_)
            b_end[ix] = e_.cpu().numpy()
            b_st[ix] = s_.cpu().numpy()
        torch.cuda.synchronize()
        t_gpu += time.time() - t0
        recon = None
        if args.recon == "gpu-gridfill":
            # gall is x-fastest over the global seed lattice, so it is the dense
            # lattice lag_gridfill expects
            tg = time.time()
            ok = torch.from_numpy(b_st == 0).to(torch.uint8).cuda()
            vals = torch.from_numpy(np.where((b_st == 0)[:, None], b_end, 0.0)).cuda()
            out, filled = P.lag_gridfill(vals, ok, dims[:g.dim])
            recon = (out.cpu().numpy(), filled.cpu().numpy().astype(bool))
            t_fill += time.time() - tg
            if it == 0:
                lat = gall[:, :g.dim] // stride
                ref, ref_in = metrics.grid_fill(lat, b_end, b_st == 0, b_st != 0)
                assert np.array_equal(recon[1] & (b_st != 0), ref_in), "gpu gridfill mask != oracle"
                assert np.array_equal(recon[0][ref_in], ref[ref_in]), "gpu gridfill != oracle (bitwise)"
        t1 = time.time()
        r = metrics.agreement(g, gall, start.cpu().numpy(), b_end, b_st, m_end.cpu().numpy(),
                              m_st.cpu().numpy(), stride, method=args.recon, recon=recon)
        t_cpu += time.time() - t1
        r["interval"] = it
        per.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    C = metrics.cell_side(g)
    Ls = [r["L"] for r in per]
    gmax, amax = metrics.max_l2_stats([r["max_l2"] for r in per])
    out = {
        "config": cfg["name"], "grid": list(g.nodes), "layout": list(cfg["layout"]), "stride": stride,
        "interval": I, "intervals": args.intervals, "cell_side_C": C,
        "total_average_L2": float(np.mean(Ls)),
        "accuracy_pct": float(np.mean([r["accuracy"] for r in per])),
        "accuracy_pct_paper_style": metrics.paper_printed_accuracy(float(np.mean(Ls)), C),
        "greatest_max_L2": gmax, "average_max_L2": amax,
        "discarded_pct": 100.0 * float(np.mean([r["discarded"] / r["seeded"] for r in per])),
        "excluded_outside_hull": int(sum(r["excluded"] for r in per)),
        "compared": int(sum(r["compared"] for r in per)),
        "gpu_seconds": t_gpu, "cpu_seconds": t_cpu, "cpu_cores": os.cpu_count(),
        "gpu_gridfill_seconds": t_fill if args.recon == "gpu-gridfill" else None,
        "method": "BTO: one context per block on one GPU; COMM map: single-block run (== decomposed COMM "
                  "bitwise); holes reconstructed by " + ("Qhull-QJ Delaunay + barycentric over valid seeds in "
                  "hole-band tiles (P:267-274)" if args.recon == "delaunay" else
                  "GridFill along lattice axes (Eq. 2, SPEC.md:323-331)" +
                  (" on the GPU (lag_gridfill)" if args.recon == "gpu-gridfill" else "")),
        "reconstruction": args.recon,
        "per_interval": [{k: r[k] for k in ("interval", "L", "max_l2", "accuracy", "discarded", "holes", "excluded")}
                         for r in per],
    }
    print(json.dumps(out), flush=True)
    if args.save:
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        tag = args.tag or f"{cfg['name']}_i{I}_{args.recon}"
        json.dump(out, open(os.path.join(ROOT, "profiles", f"agreement_{tag}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
