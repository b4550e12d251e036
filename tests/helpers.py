"""Shared test drivers: run the same seeded inputs through the CUDA path
(via the C ABI binding) and through the fp64 oracle, and compare them with
the north-star acceptance rule:

  * end positions: |Delta_a| / h_a <= 1e-4 for every particle VALID in both;
    terminated particles also keep their pre-step position within 1e-4;
  * flags: equal, except for particles whose oracle trajectory passes within
    1e-5 cells of a block face or global face (the excuse band, reading R14).
"""
from __future__ import annotations

import numpy as np

import lag_inputs as L

POS_TOL_CELLS = 1e-4
EXCUSE_CELLS = 1e-5


def global_slices(cfg, ncycles, t0_cycle=0):
    g = cfg["grid"]
    return [L.field_at_nodes(cfg["field"], g, (t0_cycle + k) * cfg["dt"]) for k in range(ncycles + 1)]


def oracle_block(cfg, block, slices, stride, mode, g_seeds=None):
    import oracle
    return oracle.run_interval(cfg["grid"], block.lo, block.hi, stride, slices, cfg["dt"],
                               mode=mode, g_seeds=g_seeds, faces=(block.lo, block.hi))


def gpu_block(cfg, block, slices, stride, mode=0, ghost=0, host=False, device=0,
              stream=None, extract_flags=0, term_cycle=False, same_tensor=None):
    """Run one interval of one block on the GPU through the C ABI.  Returns
    (start, end, status) as numpy arrays plus the Context stats."""
    import torch
    import paper_2004_02003_b200 as P
    g = cfg["grid"]
    bs = [L.cut_block_slice(V, g, block, ghost) for V in slices]
    if host:
        dev = [torch.from_numpy(np.ascontiguousarray(b)).pin_memory() for b in bs]
    else:
        dev = [torch.from_numpy(np.ascontiguousarray(b)).to(f"cuda:{device}") for b in bs]
    s = stream if stream is not None else torch.cuda.current_stream(device)
    pc = P.make_config(g.dim, g.nodes, g.origin, g.spacing, block.lo, block.hi, mode=mode,
                       ghost=ghost, device=device, stream=s.cuda_stream)
    ctx = P.Context(pc)
    try:
        n = ctx.seed(stride)
        for k in range(len(dev) - 1):
            if same_tensor is not None:          # frozen snapshot: v_t and v_t1 are one array
                ctx.advect(dev[k], dev[k] if same_tensor else dev[k + 1], cfg["dt"])
            else:
                ctx.advect(dev[k], dev[k + 1], cfg["dt"])
        start = torch.empty((n, g.dim), dtype=torch.float64, device=f"cuda:{device}")
        end = torch.empty_like(start)
        status = torch.empty((n,), dtype=torch.uint8, device=f"cuda:{device}")
        tc = torch.empty((n,), dtype=torch.int32, device=f"cuda:{device}") if term_cycle else None
        ctx.extract(start, end, status, flags=extract_flags, term_cycle=tc)
        st = ctx.stats()
        if term_cycle:
            st = dict(st, term_cycle=tc.cpu().numpy())
    finally:
        ctx.close()
    return start.cpu().numpy(), end.cpu().numpy(), status.cpu().numpy(), st


def compare(cfg, orc, start, end, status, label=""):
    """Assert the acceptance rule; return a summary dict."""
    g = cfg["grid"]
    h = np.array(g.spacing[:g.dim])
    assert start.shape == orc.start.shape, (label, start.shape, orc.start.shape)
    np.testing.assert_allclose(start, orc.start, rtol=0, atol=1e-12 * max(1.0, np.abs(orc.start).max()))
    same = status == orc.status
    excused = orc.min_face < EXCUSE_CELLS
    bad = ~same & ~excused
    assert not bad.any(), (label, "flag mismatch outside the excuse band",
                           int(bad.sum()), np.nonzero(bad)[0][:10],
                           status[bad][:10], orc.status[bad][:10], orc.min_face[bad][:10])
    cmp = same
    err = np.abs(end[cmp] - orc.pos[cmp]) / h
    worst = float(err.max()) if err.size else 0.0
    assert worst <= POS_TOL_CELLS, (label, "position error (cells)", worst,
                                    np.unravel_index(np.argmax(err), err.shape))
    return dict(n=int(status.size), valid=int((orc.status == 0).sum()),
                term=int((orc.status == 1).sum()), exit=int((orc.status == 2).sum()),
                flag_mismatch_excused=int((~same).sum()), max_err_cells=worst)
