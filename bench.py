#!/usr/bin/env python
"""Benchmark: in situ Lagrangian flow-map extraction (arXiv 2004.02003) on B200.

Metric (BASELINE.json): particle-steps/s at 1/2/4/8 B200 (BTO vs comm), % of
the memory roofline, flow-map agreement %.

Workload: C5 — ABC flow, 128^3 nodes per GPU (weak scaling, layouts (1,1,1),
(2,1,1), (2,2,1), (2,2,2)), one seed per node (2,097,152 particles per GPU),
interval 25.  A "step" is one interval: lag_seed + 25 x lag_advect_cycle +
lag_extract (every §8(a) row).  value = particle-steps of all ranks / max-over-
ranks device time of the step (CUDA events on the launching stream).  L2 is
flushed (256 MB write) before every cycle, outside the timed events.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lag|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "particle-steps/s at 1/2/4/8 B200 (BTO vs comm); % of mem roofline; flow-map agree %"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lag", choices=["lag", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-comm", action="store_true", help="skip the comm-baseline arm")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C3 (stride-2) line")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--warm-l2", action="store_true", help="do not flush L2 between cycles")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed only for process groups)

def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _coll_device():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def broadcast_bytes(b, world, rank):
    if world == 1:
        return b
    import torch.distributed as dist
    obj = [b if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    """NVML polling (2 ms) of SM clocks and clock-event reasons during the
    timed region (the B200_PROFILING.md clocks line, at a rate that resolves
    a region of a few tens of ms)."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, cuda_index):
        self.cuda_index = cuda_index
        self.sm, self.mask = [], 0
        self.stop_flag = False
        self.handle = None

    def start(self):
        try:
            import pynvml
            import torch
            self.nv = pynvml
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            try:
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.cuda_index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
            self.handle = None

    def _poll(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                self.mask |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self.handle is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_flag = True
        self.thread.join(timeout=1)
        reasons = sorted(k for k, v in self.REASONS.items()
                         if hasattr(self.nv, v) and self.mask & getattr(self.nv, v))
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_sm, "reasons": reasons, "samples": len(self.sm),
                "source": "NVML every 2 ms during the timed region"}


# ---------------------------------------------------------------------------
# the product arm

class Arm:
    """One block of the weak-scaling layout on this rank, driven through the
    C ABI binding (paper_2004_02003_b200)."""

    def __init__(self, cfg, rank, world, mode, nccl_id=None, host=False, exchange=0):
        import torch
        import lag_inputs as L
        import paper_2004_02003_b200 as P
        self.P = P
        self.cfg = cfg
        g = cfg["grid"]
        self.block = L.decompose(g, cfg["layout"])[rank]
        self.ghost = 1 if mode == P.LAG_COMM and world > 1 else 0     # no neighbour, no ghost layers
        self.interval = cfg["interval"]
        self.stream = torch.cuda.current_stream()
        lo = [self.block.lo[a] - self.ghost if a < g.dim else 0 for a in range(3)]
        ext = L.block_slice_extent(g, self.block, self.ghost)
        hi = [lo[a] + ext[a] for a in range(3)]
        # one interval's slices, generated on the device (fp64 -> fp32), untimed
        self.slices = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=lo, hi=hi,
                                        device="cuda", backend="torch").contiguous()
                       for k in range(self.interval + 1)]
        self.slice_bytes = self.slices[0].numel() * 4
        if host:
            self.slices = [s.cpu().pin_memory() for s in self.slices]
        pc = P.make_config(g.dim, g.nodes, g.origin, g.spacing, self.block.lo, self.block.hi,
                           mode=mode, ghost=self.ghost, device=torch.cuda.current_device(),
                           rank=rank, nranks=world if mode == P.LAG_COMM else 1,
                           layout=cfg["layout"] if mode == P.LAG_COMM else (1, 1, 1),
                           nccl_id=nccl_id, stream=self.stream.cuda_stream, exchange=exchange)
        self.ctx = P.Context(pc)
        self.n = self.ctx.seed(cfg["stride"])
        dev = "cpu" if host else "cuda"
        kw = dict(pin_memory=True) if host else {}
        self.start = torch.empty((self.n, g.dim), dtype=torch.float64, device=dev, **kw)
        self.end = torch.empty((self.n, g.dim), dtype=torch.float64, device=dev, **kw)
        self.status = torch.empty((self.n,), dtype=torch.uint8, device=dev, **kw)


def run_arm(arm, steps, flush, timed=True):
    """Run `steps` intervals; returns per-piece event times (ms) and the
    particle-steps done (from the library's device counters)."""
    import torch
    P = arm.P
    s = arm.stream
    t_adv, t_other, psteps = [], [], 0
    st0 = arm.ctx.stats()["particle_steps"]
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if flush is not None:
            flush.zero_()
        e0.record(s)
        arm.ctx.seed(arm.cfg["stride"])
        e1.record(s)
        pieces = [(e0, e1)]
        advs = []
        for c in range(arm.interval):
            if flush is not None:
                flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(s)
            arm.ctx.advect(arm.slices[c], arm.slices[c + 1], arm.cfg["dt"])
            a1.record(s)
            advs.append((a0, a1))
        if flush is not None:
            flush.zero_()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(s)
        # LAG_ASYNC: the write cycle is enqueued without a host round trip, so
        # the device events time only the library's kernels
        arm.ctx.extract(arm.start, arm.end, arm.status, flags=P.LAG_NO_RESEED | P.LAG_ASYNC)
        x1.record(s)
        pieces.append((x0, x1))
        torch.cuda.synchronize()
        t_adv.append(sum(a.elapsed_time(b) for a, b in advs))
        t_other.append(sum(a.elapsed_time(b) for a, b in pieces))
    st1 = arm.ctx.stats()
    if st1["device_error"] != 0:          # latched during the asynchronous write cycles
        raise RuntimeError(f"latched device error {st1['device_error']} in the timed intervals")
    psteps = st1["particle_steps"] - st0
    return t_adv, t_other, psteps


def run_e2e(cfg, rank, world, steps, warmup):
    """Same metric through the public C ABI with HOST buffers: pinned host
    slices staged by the library (H2D inside the timed region) and the flow
    map returned into pinned host arrays (D2H inside the timed region).  The
    K steps run back to back as a user's loop would (the write cycle is
    enqueued with LAG_ASYNC into one of two pinned output sets, so step k's
    flow-map copy overlaps step k+1's slice uploads); the wall clock brackets
    all K steps with a synchronize on both sides."""
    import torch
    import paper_2004_02003_b200 as P
    arm = Arm(cfg, rank, world, P.LAG_BTO, host=True)
    h2d = arm.slice_bytes * (arm.interval + 1)
    d2h = arm.start.numel() * 8 + arm.end.numel() * 8 + arm.status.numel()
    outs = [(arm.start, arm.end, arm.status),
            tuple(torch.empty_like(t, pin_memory=True) for t in (arm.start, arm.end, arm.status))]

    def run(k0, n):
        for it in range(k0, k0 + n):
            o = outs[it % 2]
            arm.ctx.seed(cfg["stride"])
            for c in range(arm.interval):
                arm.ctx.advect(arm.slices[c], arm.slices[c + 1], cfg["dt"])
            arm.ctx.extract(o[0], o[1], o[2], flags=P.LAG_NO_RESEED | P.LAG_ASYNC)

    run(0, warmup)
    torch.cuda.synchronize()
    st0 = arm.ctx.stats()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(warmup, steps)
    torch.cuda.synchronize()
    dt = allreduce_max(time.perf_counter() - t0, world)
    st1 = arm.ctx.stats()
    if st1["device_error"] != 0:
        raise RuntimeError(f"latched device error {st1['device_error']} in the e2e steps")
    total_ps = allreduce_sum(st1["particle_steps"] - st0["particle_steps"], world)
    arm.ctx.close()
    return {"value": total_ps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / steps,
            "timing": "wall clock around K back-to-back steps (synchronize before and after), max over ranks"}


def algorithmic_bytes(name, psteps, cycles, slice_bytes, interval=None):
    """Algorithmic bytes of `cycles` advect launches: 32 B per particle-step
    (float4 read + write) + the slice sectors the method's stage gathers touch
    per cycle (profiles/algbytes.json, written by scripts/algbytes.py from the
    oracle's touched-node maps; both whole slices if absent).  The sampled
    cycles are averaged over an interval with the first cycle (particles on
    their seed nodes) weighted 1/interval."""
    vel = 2.0 * slice_bytes
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "algbytes.json")))[name]
        per = {c["cycle"]: 32.0 * (c["sectors_v_t"] + c["sectors_v_t1"]) for c in d["cycles"]}
        later = [v for k, v in per.items() if k > 0]
        I = interval or d.get("interval") or 25
        if 0 in per and later:
            vel = (per[0] + (I - 1) * float(np.mean(later))) / I
        else:
            vel = float(np.mean(list(per.values())))
    except Exception:
        pass
    return 32.0 * psteps + cycles * vel


def measure_secondary(name, rank, world, steps, warmup, flush):
    """BTO throughput + roofline of another per-GPU workload (C3: stride 2,
    the HBM-heavy configuration)."""
    import torch
    import lag_inputs as L
    import paper_2004_02003_b200 as P
    cfg = L.make_config(name, nranks=world)
    arm = Arm(cfg, rank, world, P.LAG_BTO)
    run_arm(arm, warmup, flush)
    barrier(world)
    torch.cuda.synchronize()
    t_adv, t_other, psteps = run_arm(arm, steps, flush)
    adv_ms, dev_ms = sum(t_adv), sum(t_adv) + sum(t_other)
    dev_ms_max = allreduce_max(dev_ms, world)
    total_ps = allreduce_sum(psteps, world)
    cycles = steps * arm.interval
    alg = algorithmic_bytes(name, psteps, cycles, arm.slice_bytes, arm.interval)
    peak, _ = measured_peak()
    ach = alg / (adv_ms / 1e3) / 1e9
    out = {"workload": f"{name}: {cfg['field'].kind} field, {list(L.block_slice_extent(cfg['grid'], arm.block, 0))} "
                       f"slice nodes per GPU, stride {cfg['stride']}, {arm.n} particles/GPU, interval {cfg['interval']}",
           "value": total_ps / (dev_ms_max / 1e3), "unit": UNIT, "ms_per_step": dev_ms_max / steps,
           "ms_per_cycle": allreduce_max(adv_ms, world) / cycles,
           "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                        "alg_bytes_per_launch": alg / cycles}}
    arm.ctx.close()
    return out


def measure_c2(steps, warmup, flush):
    """configs[1] on one GPU: C2 = ABC 128^3 as 8 blocks (2x2x2), stride 1,
    interval 25, BTO vs COMM.  BTO: 8 contexts, one stream each.  COMM: the
    same 8 blocks as one LAG_XCHG_LOCAL group (ghost layers copied from the
    neighbours' slices, hand-offs appended from their slots every cycle,
    return to origin at the write cycle), one stream each.  Each arm's
    interval is captured as three CUDA graphs (seed, the 25 cycles, the write
    cycle) and replayed: at 262144 particles per block the cycle is
    launch-bound, which the graph removes.  L2 is flushed
    before every interval (the whole C2 working set, ~86 MB, fits in L2)."""
    import torch
    import lag_inputs as L
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2")
    g = cfg["grid"]
    I = cfg["interval"]
    blocks = L.decompose(g, cfg["layout"])
    main_s = torch.cuda.Stream()          # graphs are captured on a non-default stream

    def build(mode):
        ghost = 1 if mode == P.LAG_COMM else 0
        streams = [torch.cuda.Stream() for _ in blocks]
        cfgs, slices = [], []
        for b, st in zip(blocks, streams):
            lo = [b.lo[a] - ghost for a in range(3)]
            ext = L.block_slice_extent(g, b, ghost)
            hi = [lo[a] + ext[a] for a in range(3)]
            slices.append([L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=lo, hi=hi, device="cuda",
                                            backend="torch").contiguous() for k in range(I + 1)])
            cfgs.append(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=mode,
                                      ghost=ghost, rank=b.rank if mode == P.LAG_COMM else 0,
                                      nranks=len(blocks) if mode == P.LAG_COMM else 1,
                                      layout=cfg["layout"] if mode == P.LAG_COMM else (1, 1, 1),
                                      stream=st.cuda_stream,
                                      exchange=P.LAG_XCHG_LOCAL if mode == P.LAG_COMM else 0))
        if mode == P.LAG_COMM:
            grp = P.LocalGroup(cfgs)
            ctxs = grp.blocks
        else:
            grp = None
            ctxs = [P.Context(c) for c in cfgs]
        ns = [c.seed(cfg["stride"]) for c in ctxs]
        outs = [(torch.empty((n, 3), dtype=torch.float64, device="cuda"),
                 torch.empty((n, 3), dtype=torch.float64, device="cuda"),
                 torch.empty((n,), dtype=torch.uint8, device="cuda")) for n in ns]
        torch.cuda.synchronize()

        def fork():
            ev = torch.cuda.Event()
            ev.record(main_s)
            for st in streams:
                st.wait_event(ev)

        def join():
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                main_s.wait_event(ev)

        def seed_all():
            for c in ctxs:
                c.seed(cfg["stride"])

        def cycles_all():
            for k in range(I):
                for c, sl in zip(ctxs, slices):
                    c.advect(sl[k], sl[k + 1], cfg["dt"])

        def extract_all():
            for c, o in zip(ctxs, outs):
                c.extract(*o, flags=P.LAG_NO_RESEED | P.LAG_ASYNC)

        graphs = []
        for fn in (seed_all, cycles_all, extract_all):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=main_s):
                fork()
                fn()
                join()
            graphs.append(gr)
        torch.cuda.synchronize()
        return dict(ctxs=ctxs, grp=grp, graphs=graphs, n=sum(ns))

    def run(arm, nsteps):
        t_int, t_cyc = [], []
        for _ in range(nsteps):
            if flush is not None:
                flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(main_s)
            arm["graphs"][0].replay()
            ev[1].record(main_s)
            arm["graphs"][1].replay()
            ev[2].record(main_s)
            arm["graphs"][2].replay()
            ev[3].record(main_s)
            torch.cuda.synchronize()
            t_int.append(ev[0].elapsed_time(ev[3]))
            t_cyc.append(ev[1].elapsed_time(ev[2]))
        return t_int, t_cyc

    res = {}
    for name, mode in (("bto", P.LAG_BTO), ("comm", P.LAG_COMM)):
        arm = build(mode)
        with torch.cuda.stream(main_s):
            run(arm, warmup)
            ps0 = sum(c.stats()["particle_steps"] for c in arm["ctxs"])
            t_int, t_cyc = run(arm, steps)
        stats = [c.stats() for c in arm["ctxs"]]
        if any(st["device_error"] for st in stats):
            raise RuntimeError(f"latched device error in the C2 {name} leg")
        ps = sum(st["particle_steps"] for st in stats) - ps0
        res[name] = {"value": ps / (sum(t_int) / 1e3), "unit": UNIT, "ms_per_step": sum(t_int) / steps,
                     "ms_per_cycle": sum(t_cyc) / steps / I,
                     "particle_steps_per_s_cycles_only": ps / (sum(t_cyc) / 1e3),
                     "discarded_last_interval": int(sum(st["term_boundary"] + st["exit_domain"] for st in stats)),
                     "sent_last_interval": int(sum(st["sent"] for st in stats)),
                     "received_last_interval": int(sum(st["received"] for st in stats))}
        if arm["grp"] is not None:
            arm["grp"].close()
        else:
            for c in arm["ctxs"]:
                c.close()
        del arm
        torch.cuda.synchronize()
    return {"workload": "C2 (configs[1]): ABC 128^3 as 8 blocks (2x2x2) on one GPU, stride 1 "
                        "(2097152 particles), interval 25; one stream per block; each interval replayed "
                        "as CUDA graphs (seed | 25 cycles | write cycle); COMM = LAG_XCHG_LOCAL",
            "bto": res["bto"], "comm": res["comm"],
            "value": res["bto"]["value"], "unit": UNIT,
            "bto_speedup_per_cycle": res["comm"]["ms_per_cycle"] / res["bto"]["ms_per_cycle"],
            "bto_speedup_step": res["comm"]["ms_per_step"] / res["bto"]["ms_per_step"],
            "l2": "flushed before every interval; the cycles of an interval run back to back"}


def measure_c4(steps, warmup, flush):
    """configs[3] per GPU: C4 = Nyx-like turbulence 512^3 as 2x2x2, block 0
    (256^3 owned nodes, 257^3 slice nodes, 203.7 MB per slice), stride 4
    (262144 particles), BTO, intervals 10 / 50 / 100 (the paper's sweep,
    P:782-783).  Roofline bytes: profiles/algbytes.json C4@<interval>."""
    import torch
    import lag_inputs as L
    import paper_2004_02003_b200 as P
    peak, _ = measured_peak()
    out = {"workload": "C4 (configs[3]): Nyx-like 64-mode turbulence, 512^3 as 2x2x2, block 0 "
                       "(257^3 slice nodes) on one GPU, stride 4 (262144 particles), BTO"}
    for I in (10, 50, 100):
        cfg = L.make_config("C4", interval=I)
        arm = Arm(cfg, 0, 1, P.LAG_BTO)
        run_arm(arm, warmup, flush)
        torch.cuda.synchronize()
        t_adv, t_other, psteps = run_arm(arm, steps, flush)
        adv_ms, dev_ms = sum(t_adv), sum(t_adv) + sum(t_other)
        cycles = steps * I
        alg = algorithmic_bytes(f"C4@{I}", psteps, cycles, arm.slice_bytes, I)
        ach = alg / (adv_ms / 1e3) / 1e9
        st = arm.ctx.stats()
        out[f"interval_{I}"] = {
            "value": psteps / (dev_ms / 1e3), "unit": UNIT, "ms_per_step": dev_ms / steps,
            "ms_per_cycle": adv_ms / cycles,
            "discarded_pct_last_interval": 100.0 * (st["term_boundary"] + st["exit_domain"]) / arm.n,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "alg_bytes_per_launch": alg / cycles}}
        arm.ctx.close()
        del arm
        torch.cuda.empty_cache()
    return out


def c1_cpu_seconds():
    """configs[0]: C1 double gyre 64x32, 2048 particles, 100 RK4 cycles in 5
    intervals of 20 — the whole run through the fp64 oracle on 1 host core and
    on all host cores (CPU seconds), and the same run on the GPU through the C
    ABI (device time)."""
    import ctypes
    import torch
    import lag_inputs as L
    import oracle
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C1")
    g = cfg["grid"]
    I, C = cfg["interval"], cfg["cycles"]
    sl = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"]) for k in range(C + 1)]
    try:
        gomp = ctypes.CDLL("libgomp.so.1")
    except OSError:
        gomp = None
    oracle.build()
    res = {}
    ncpu = os.cpu_count() or 1
    for cores in (1, ncpu):
        if gomp is not None:
            gomp.omp_set_num_threads(cores)
        t0 = time.perf_counter()
        for it in range(C // I):
            iv = oracle.Interval(g, (0, 0, 0), g.nodes, 1)
            for c in range(I):
                iv.cycle(sl[it * I + c], sl[it * I + c + 1], cfg["dt"])
        res[f"cpu_seconds_{cores}_cores"] = time.perf_counter() - t0
    if gomp is not None:
        gomp.omp_set_num_threads(ncpu)
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    # the same 100 cycles on the GPU
    s = torch.cuda.current_stream()
    dev = [torch.from_numpy(v).cuda() for v in sl]
    ctx = P.Context(P.make_config(2, g.nodes, g.origin, g.spacing, (0, 0, 0), g.nodes, stream=s.cuda_stream))
    n = ctx.seed(1)
    end = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for it in range(C // I):
        for c in range(I):
            ctx.advect(dev[it * I + c], dev[it * I + c + 1], cfg["dt"])
        ctx.extract(end=end, flags=P.LAG_ASYNC)
    e1.record(s)
    torch.cuda.synchronize()
    res["gpu_seconds"] = e0.elapsed_time(e1) / 1e3
    ctx.close()
    res.update({"workload": "C1 (configs[0]): double gyre 64x32, 1 block, 2048 particles, 100 cycles, interval 20",
                "particle_steps": 2048 * C, "host_cores": ncpu, "cpu_model": model,
                "cpu": "fp64 C oracle (OpenMP over particles), whole run incl. reseeds"})
    return res


def measured_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    p = os.path.join(ROOT, "profiles", "advect_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config)
    except Exception:
        return None


def cpu_baseline(cfg, seconds_target=10.0, max_particles=None):
    """The fp64 oracle as it stands, on the host cores, on a bounded sample of
    the same workload: the block's seeds (strided subset if max_particles)
    advanced through whole intervals (reseeded each time) until about
    `seconds_target` of CPU work has been done."""
    import lag_inputs as L
    import oracle
    g = cfg["grid"]
    block = L.decompose(g, cfg["layout"])[0]
    cores = int(os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1)))
    seeds = oracle.seeds(g, block.lo, block.hi, cfg["stride"])
    if max_particles and seeds.shape[0] > max_particles:
        seeds = seeds[:: seeds.shape[0] // max_particles][:max_particles]
    ncyc = cfg["interval"]
    sl = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"], backend="torch").numpy()
          for k in range(ncyc + 1)]
    el, psteps, intervals = 0.0, 0, 0
    while el < seconds_target and intervals < 50:
        it = oracle.Interval(g, block.lo, block.hi, cfg["stride"], g_seeds=seeds)
        t0 = time.perf_counter()
        for c in range(ncyc):
            psteps += it.active()
            it.cycle(sl[c], sl[c + 1], cfg["dt"])
        el += time.perf_counter() - t0
        intervals += 1
    return {"value": psteps / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{intervals} interval(s) of {ncyc} cycles over {seeds.shape[0]} seeds of the "
                      f"{cfg['name']} block (fp64 C oracle, OpenMP), {el:.1f} s of CPU work"}


def reference_arm(args):
    """--impl reference: the oracle on the host cores as the reference arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # rank 0 alone runs it: on all host cores (torchrun sets OMP_NUM_THREADS=1
    # per process; the OpenMP runtime reads it when the oracle library loads)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import lag_inputs as L
    cfg = L.make_config(args.config, nranks=1)
    vals = []
    budget = max(1.0, 90.0 / max(1, args.steps))
    for _ in range(max(1, args.steps)):
        vals.append(cpu_baseline(cfg, seconds_target=budget))
    v = statistics.median(x["value"] for x in vals)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{cfg['name']} ABC 128^3 block, stride 1, interval 25 (bounded sample)"},
           "cpu_baseline": {"kind": "oracle", "cores": vals[0]["cores"], "sample": vals[0]["sample"],
                            "value": v},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import lag_inputs as L
    import paper_2004_02003_b200 as P
    rank, world, local = dist_setup(args.gpus)
    cfg = L.make_config(args.config, nranks=world)
    flush = None if args.warm_l2 else torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    # ---------------- BTO (the paper's method): headline ----------------
    arm = Arm(cfg, rank, world, P.LAG_BTO)
    run_arm(arm, args.warmup, flush)
    launches0 = arm.ctx.launches()
    clk = ClockSampler(local)
    clk.start()
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t_adv, t_other, psteps = run_arm(arm, args.steps, flush)
    barrier(world)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    clocks = clk.stop()
    launches = arm.ctx.launches() - launches0
    dev_ms = sum(t_adv) + sum(t_other)
    adv_ms = sum(t_adv)
    dev_ms_max = allreduce_max(dev_ms, world)
    adv_ms_max = allreduce_max(adv_ms, world)
    total_ps = allreduce_sum(psteps, world)
    value = total_ps / (dev_ms_max / 1e3)
    # roofline of the dominant kernel (advect): algorithmic bytes per launch =
    # 32 B x active particles (float4 read + write) + the slice sectors the
    # method touches (stride 1: every node) — DESIGN.md §6
    cycles = args.steps * arm.interval
    alg_bytes = algorithmic_bytes(cfg["name"], psteps, cycles, arm.slice_bytes, arm.interval)
    achieved = alg_bytes / (adv_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    st = arm.ctx.stats()
    n_per_rank = arm.n
    arm.ctx.close()
    del arm

    # ---------------- comm baseline (Lagrangian-MPI analogue) ----------------
    # both transports; the BTO speed-up is quoted against the faster one
    comm = None
    if not args.no_comm:
      try:
        comm = {}
        transports = [("nccl", P.LAG_XCHG_NCCL)] + ([("peer", P.LAG_XCHG_PEER),
                                                     ("peer_overlap", P.LAG_XCHG_PEER_OVERLAP)] if world > 1 else [])
        for tname, xch in transports:
            nid = broadcast_bytes(P.lag_nccl_unique_id() if rank == 0 else None, world, rank) if world > 1 else None
            carm = Arm(cfg, rank, world, P.LAG_COMM, nccl_id=nid, exchange=xch)
            run_arm(carm, args.warmup, flush)
            barrier(world)
            c_adv, c_other, c_ps = run_arm(carm, args.steps, flush)
            c_ms = allreduce_max(sum(c_adv) + sum(c_other), world)
            c_total = allreduce_sum(c_ps, world)
            cst = carm.ctx.stats()
            c_cyc = allreduce_max(sum(c_adv), world) / cycles
            comm[tname] = {"value": c_total / (c_ms / 1e3), "unit": UNIT,
                           "ms_per_step": c_ms / args.steps,
                           "ms_per_cycle": c_cyc,
                           # the paper's metric: average time per cycle (advection,
                           # management, communication), write cycles excluded
                           "bto_speedup": c_cyc / (adv_ms_max / cycles),
                           "bto_speedup_step": c_ms / dev_ms_max,
                           "sent_last_interval": int(cst["sent"]),
                           "received_last_interval": int(cst["received"])}
            carm.ctx.close()
            del carm
        best = max(comm.values(), key=lambda d: d["value"])
        comm.update({"value": best["value"], "unit": UNIT, "bto_speedup": best["bto_speedup"],
                     "bto_speedup_step": best["bto_speedup_step"],
                     "exchange": "per cycle: ghost layer (G=1, faces+edges+corners) of v_t1 + particle "
                                 "hand-offs; 'nccl' = one grouped NCCL send/recv, 'peer' = kernels read / "
                                 "write the neighbours' memory over NVLink (CUDA IPC), 'peer_overlap' = "
                                 "peer with the exchange run by the first CTAs of the advect kernel while "
                                 "the other CTAs advect the ghost-free tiles; value/speedup = fastest; "
                                 "bto_speedup = per-cycle time ratio (write cycles excluded, P:365-367), "
                                 "bto_speedup_step = whole-interval ratio"})
      except Exception as exc:        # the headline BTO line must still print
        comm = {"error": repr(exc)[:300]}

    secondary = None
    if not args.no_secondary:
        try:
            secondary = measure_secondary("C3", rank, world, max(2, args.steps // 2), 2, flush)
        except Exception as exc:
            secondary = {"error": repr(exc)[:300]}

    c2 = None
    if world == 1 and not args.no_secondary:
        try:
            c2 = measure_c2(max(2, args.steps // 2), 2, flush)
        except Exception as exc:
            c2 = {"error": repr(exc)[:300]}

    c4 = None
    if world == 1 and not args.no_secondary:
        try:
            c4 = measure_c4(1, 1, flush)
        except Exception as exc:
            c4 = {"error": repr(exc)[:300]}

    c1 = None
    if world == 1 and not args.no_cpu:
        try:
            c1 = c1_cpu_seconds()
        except Exception as exc:
            c1 = {"error": repr(exc)[:300]}

    e2e = None
    if not args.no_e2e:
        try:
            e2e = run_e2e(cfg, rank, world, max(2, args.steps // 2), 1)
        except Exception as exc:
            e2e = {"error": repr(exc)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(cfg)
        except Exception as exc:
            cpu = {"error": repr(exc)[:300]}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg['name']}: ABC flow 128^3 nodes per GPU, 1 seed/node "
                                   f"({n_per_rank} particles/GPU), interval {cfg['interval']}, BTO",
                       "layout": list(cfg["layout"]), "global_nodes": list(cfg["grid"].nodes),
                       "particles_per_gpu": n_per_rank, "cycles_per_step": arm_interval(cfg),
                       "step": "lag_seed + interval x lag_advect_cycle + lag_extract",
                       "l2": "warm (no flush)" if args.warm_l2 else
                             "flushed (256 MB write) before every cycle, outside the timed events",
                       "wall_s_timed_region": wall,
                       "ms_per_cycle": adv_ms_max / cycles,
                       "discarded_last_interval": int(st["term_boundary"] + st["exit_domain"]),
                       "parallelism": f"dp{world} (one block per GPU, no collective)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(cfg["name"]),
                         "kernel": "advect_kernel<3,true,false>", "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes / cycles,
                         "kernel_share_of_step": adv_ms / dev_ms},
            "comm": comm,
            "secondary": secondary,
            "c2": c2,
            "c4": c4,
            "c1_cpu_seconds": c1,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def arm_interval(cfg):
    return cfg["interval"]


if __name__ == "__main__":
    main()
