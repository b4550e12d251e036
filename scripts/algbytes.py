"""Algorithmic bytes per cycle of the advect kernel, from the oracle's
definition of the method:

  B_cycle = 32 B x N_active (float4 record read + write)
          + 32 B x (#unique 32-byte sectors of v_t and v_t1 the cycle's RK4
            stage gathers touch: stage 1 reads only v_t, stage 4 only v_t1)

The touched-node maps come from oracle.orc_cycle's instrumentation; sectors
are counted on the caller's AoS fp32 layout (12 B per node in 3-D).  Writes
profiles/algbytes.json, read by bench.py.  Calls only oracle/ and lag_inputs/.

  python scripts/algbytes.py [configs...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lag_inputs as L  # noqa: E402
import oracle  # noqa: E402


def sectors(mask: np.ndarray, node_bytes: int) -> int:
    """Unique 32 B sectors covered by the touched nodes of one slice."""
    idx = np.nonzero(mask.ravel())[0].astype(np.int64)
    if idx.size == 0:
        return 0
    first = (idx * node_bytes) // 32
    last = (idx * node_bytes + node_bytes - 1) // 32
    return int(np.unique(np.concatenate([first, last])).size)


def measure(name, cycles=(0, 5, 12, 24)):
    cfg = L.make_config(name)
    g = cfg["grid"]
    b = L.decompose(g, cfg["layout"])[0]
    nb = 4 * g.dim
    it = oracle.Interval(g, b.lo, b.hi, cfg["stride"])
    slice_nodes = int(np.prod([min(b.hi[a] + 1, g.nodes[a]) - b.lo[a] for a in range(g.dim)]))
    out = []
    V0 = L.field_at_nodes(cfg["field"], g, 0.0, backend="torch").numpy()
    for c in range(max(cycles) + 1):
        V1 = L.field_at_nodes(cfg["field"], g, (c + 1) * cfg["dt"], backend="torch").numpy()
        touched = np.zeros(g.nodes[::-1], dtype=np.uint8) if c in cycles else None
        n_active = it.active()
        it.cycle(V0, V1, cfg["dt"], touched=touched)
        if touched is not None:
            s0 = sectors(touched & 1, nb)
            s1 = sectors(touched & 2, nb)
            full = (slice_nodes * nb + 31) // 32
            out.append(dict(cycle=c, n_active=n_active, sectors_v_t=s0, sectors_v_t1=s1,
                            slice_sectors=full, bytes=32 * n_active + 32 * (s0 + s1),
                            bytes_per_particle_step=(32 * n_active + 32 * (s0 + s1)) / max(1, n_active)))
            print(name, out[-1], flush=True)
        V0 = V1
    return dict(config=name, stride=cfg["stride"], block=[list(b.lo), list(b.hi)], cycles=out,
                mean_bytes_per_particle_step=float(np.mean([o["bytes_per_particle_step"] for o in out])),
                mean_touched_fraction=float(np.mean([(o["sectors_v_t"] + o["sectors_v_t1"]) /
                                                     (2 * o["slice_sectors"]) for o in out])))


def measure_c4(interval):
    """C4 (Nyx-like 512^3 as 2x2x2, stride 4): block 0 = nodes [0, 256)^3.  A BTO
    particle of block 0 gathers only nodes [0, 256]^3 (samples beyond the
    block face stop before their gather), so the oracle runs on that
    257^3 sub-grid with the real field values; the touched maps are those of
    the full grid.  Samples cycles 0, mid and last of an interval."""
    cfg = L.make_config("C4")
    g = cfg["grid"]
    sub = L.Grid(3, (257, 257, 257), g.origin, g.spacing)
    nb = 12
    it = oracle.Interval(sub, (0, 0, 0), (256, 256, 256), cfg["stride"])
    want = sorted({0, interval // 2, interval - 1})
    out = []
    V0 = L.field_at_nodes(cfg["field"], g, 0.0, hi=(257, 257, 257), backend="torch").numpy()
    for c in range(interval):
        V1 = L.field_at_nodes(cfg["field"], g, (c + 1) * cfg["dt"], hi=(257, 257, 257), backend="torch").numpy()
        touched = np.zeros((257, 257, 257), dtype=np.uint8) if c in want else None
        n_active = it.active()
        it.cycle(V0, V1, cfg["dt"], touched=touched)
        if touched is not None:
            s0 = sectors(touched & 1, nb)
            s1 = sectors(touched & 2, nb)
            full = (257 ** 3 * nb + 31) // 32
            out.append(dict(cycle=c, n_active=n_active, sectors_v_t=s0, sectors_v_t1=s1,
                            slice_sectors=full, bytes=32 * n_active + 32 * (s0 + s1),
                            bytes_per_particle_step=(32 * n_active + 32 * (s0 + s1)) / max(1, n_active)))
            print("C4", interval, out[-1], flush=True)
        V0 = V1
    return dict(config="C4", interval=interval, stride=cfg["stride"], block=[[0, 0, 0], [256, 256, 256]],
                cycles=out, discarded=int(it.n - it.active()), seeded=int(it.n),
                mean_bytes_per_particle_step=float(np.mean([o["bytes_per_particle_step"] for o in out])),
                mean_touched_fraction=float(np.mean([(o["sectors_v_t"] + o["sectors_v_t1"]) /
                                                     (2 * o["slice_sectors"]) for o in out])))


def main():
    names = sys.argv[1:] or ["C5", "C3"]
    path = os.path.join(ROOT, "profiles", "algbytes.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for n in names:
        if n.startswith("C4@"):
            res[n] = measure_c4(int(n[3:]))
            json.dump(res, open(path, "w"), indent=1)
            continue
        res[n] = measure(n)
    res["_source"] = ("scripts/algbytes.py: oracle touched-node maps (stage gathers of the method), "
                      "unique 32 B sectors of the AoS fp32 slices + 32 B per active particle")
    json.dump(res, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
