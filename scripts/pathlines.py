"""Pathline accuracy from stitched flow maps vs ground truth (SURVEY.md
§8(f)2; the paper's pathline comparison).

All compute runs on the GPU through the C ABI:
  * BTO flow maps of K successive intervals of I cycles at stride s, one
    context per block of the layout, holes filled by lag_gridfill;
  * COMM flow maps of the same intervals: a single block over the whole
    domain, which equals the decomposed COMM run bitwise; its global-domain
    exits are GridFilled like BTO's holes;
  * both stitched by lag_stitch from the nodes between the stride-s seeds
    (all coordinates odd multiples of s/2 when s is even; else a node sample);
  * ground truth: one block, stride 1, one interval of K*I cycles. This is
    full-resolution RK4 with no resets.
Prints one JSON line with the error in cells (mean / median / p99 / max),
truncation counts and kernel times; --save writes profiles/pathlines_<tag>.json.

  python scripts/pathlines.py [config] [--scale N] [--K 4] [--interval I] [--stride S] [--save]
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


def run_blocks(cfg, blocks, stride, t0_cycle, ncycles, dims_l, sp_l):
    """One interval on every block (device slices); returns lattice ends [n, d] and valid [n]."""
    g = cfg["grid"]
    n = int(np.prod(dims_l))
    ends = torch.full((n, g.dim), float("nan"), dtype=torch.float64, device="cuda")
    valid = torch.zeros((n,), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    ctxs = [P.Context(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi, stream=s.cuda_stream))
            for b in blocks]
    ns = [c.seed(stride) for c in ctxs]
    ext = [L.block_slice_extent(g, b, 0) for b in blocks]
    for k in range(ncycles):
        t = (t0_cycle + k) * cfg["dt"]
        V0 = L.field_at_nodes(cfg["field"], g, t, device="cuda", backend="torch")
        V1 = L.field_at_nodes(cfg["field"], g, t + cfg["dt"], device="cuda", backend="torch")
        for c, b, e in zip(ctxs, blocks, ext):
            sl = tuple(slice(b.lo[a], b.lo[a] + e[a]) for a in (2, 1, 0))
            c.advect(V0[sl].contiguous(), V1[sl].contiguous(), cfg["dt"])
    for c, nn in zip(ctxs, ns):
        st = torch.empty((nn, g.dim), dtype=torch.float64, device="cuda")
        en = torch.empty_like(st)
        ss = torch.empty((nn,), dtype=torch.uint8, device="cuda")
        c.extract(st, en, ss)
        q = torch.round((st - torch.tensor(g.origin[:g.dim], device="cuda", dtype=torch.float64))
                        / torch.tensor(sp_l, device="cuda", dtype=torch.float64)).long()
        flat = q[:, 0] + dims_l[0] * (q[:, 1] + (dims_l[1] * q[:, 2] if g.dim == 3 else 0))
        ends[flat] = en
        valid[flat] = (ss == 0).to(torch.uint8)
        c.close()
    return ends, valid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--K", type=int, default=4)
    ap.add_argument("--interval", type=int, default=None)
    ap.add_argument("--stride", type=int, default=2)
    ap.add_argument("--layout", default=None)
    ap.add_argument("--save", action="store_true")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    cfg = L.make_config(args.config, scale=args.scale, interval=args.interval)
    if args.layout:
        cfg["layout"] = tuple(int(x) for x in args.layout.split(","))
    g = cfg["grid"]
    I, K, s = cfg["interval"], args.K, args.stride
    dims_l = tuple(int(-(-g.nodes[a] // s)) for a in range(g.dim))
    sp_l = tuple(s * g.spacing[a] for a in range(g.dim))
    blocks = L.decompose(g, cfg["layout"])
    whole = [L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)]
    maps = {"bto": [], "comm": []}
    t_fill = 0.0
    for k in range(K):
        e, v = run_blocks(cfg, blocks, s, k * I, I, dims_l, sp_l)
        torch.cuda.synchronize()
        t0 = time.time()
        f, _ = P.lag_gridfill(e, v, dims_l)
        t_fill += time.time() - t0
        maps["bto"].append(f)
        # domain exits are invalid in both maps; both are GridFilled the same
        # way, so the comparison isolates BTO's block-boundary holes
        e2, v2 = run_blocks(cfg, whole, s, k * I, I, dims_l, sp_l)
        f2, _ = P.lag_gridfill(e2, v2, dims_l)
        maps["comm"].append(f2)
    # ground truth at stride 1 over the whole run
    gt_e, gt_v = run_blocks(cfg, whole, 1, 0, K * I, tuple(g.nodes[:g.dim]), tuple(g.spacing[:g.dim]))
    nodes = np.indices(tuple(g.nodes[:g.dim])[::-1]).reshape(g.dim, -1)[::-1].T
    if s % 2 == 0:
        sel = ((nodes % s) == s // 2).all(axis=1)
    else:
        sel = np.random.default_rng(0).random(nodes.shape[0]) < 0.05
    sel &= gt_v.cpu().numpy().astype(bool)
    starts = torch.from_numpy(np.asarray(g.origin[:g.dim]) + nodes[sel] * np.asarray(g.spacing[:g.dim])).cuda()
    truth = gt_e.cpu().numpy()[sel]
    out = {"config": cfg["name"], "grid": list(g.nodes), "layout": list(cfg["layout"]), "stride": s,
           "interval": I, "K": K, "queries": int(sel.sum()), "gridfill_seconds": t_fill}
    for name, ms in maps.items():
        ends = torch.stack(ms).contiguous()
        vmask = (~torch.isnan(ends).any(dim=2)).to(torch.uint8).contiguous()
        torch.cuda.synchronize()
        t0 = time.time()
        path, st = P.lag_stitch(ends, starts, dims_l, g.origin[:g.dim], sp_l, valid=vmask)
        torch.cuda.synchronize()
        dt = time.time() - t0
        st = st.cpu().numpy()
        ok = st == 0
        err = np.linalg.norm(path.cpu().numpy()[ok, K] - truth[ok], axis=1) / min(g.spacing[:g.dim])
        out[name] = {"complete": int(ok.sum()), "out_of_hull": int((st == 1).sum()),
                     "invalid_flow": int((st == 2).sum()), "stitch_seconds": dt,
                     "err_cells_mean": float(err.mean()), "err_cells_median": float(np.median(err)),
                     "err_cells_p99": float(np.quantile(err, 0.99)), "err_cells_max": float(err.max())}
    print(json.dumps(out), flush=True)
    if args.save:
        tag = args.tag or f"{cfg['name']}_s{s}_i{I}_K{K}"
        json.dump(out, open(os.path.join(ROOT, "profiles", f"pathlines_{tag}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
