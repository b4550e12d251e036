"""Thin ctypes binding of liblag (include/lag.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback — if liblag.so is missing the import fails loudly.

Functions carry the C names (lag_init, lag_seed, lag_advect_cycle,
lag_extract, lag_stats, lag_destroy, lag_last_error, lag_nccl_unique_id);
a non-zero lag_status raises LagError.  Array arguments may be torch tensors
(device or host), numpy arrays, or raw integer addresses.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LAG_LIB") or os.path.join(HERE, "liblag.so")

LAG_OK, LAG_EINVAL, LAG_ESTATE, LAG_EEMPTY, LAG_ENOMEM = 0, -1, -2, -3, -4
LAG_ECUDA, LAG_ENCCL, LAG_EOVERFLOW, LAG_EGHOST, LAG_ENONFINITE = -5, -6, -7, -8, -9
LAG_BTO, LAG_COMM = 0, 1
LATCHED = (-7, -8, -9)       # async conditions lag_extract reports after writing its outputs
LAG_XCHG_NCCL, LAG_XCHG_PEER, LAG_XCHG_PEER_OVERLAP, LAG_XCHG_LOCAL = 0, 1, 2, 3
LAG_VALID, LAG_TERM_BOUNDARY, LAG_EXIT_DOMAIN = 0, 1, 2
LAG_ABI_VERSION = 3          # include/lag.h
LAG_NO_RESEED = 1
LAG_ASYNC = 2
STATUS_NAMES = {0: "LAG_OK", -1: "LAG_EINVAL", -2: "LAG_ESTATE", -3: "LAG_EEMPTY",
                -4: "LAG_ENOMEM", -5: "LAG_ECUDA", -6: "LAG_ENCCL", -7: "LAG_EOVERFLOW",
                -8: "LAG_EGHOST", -9: "LAG_ENONFINITE"}

# every symbol include/lag.h declares
EXPORTS = ("lag_init", "lag_seed", "lag_advect_cycle", "lag_extract", "lag_extract_ex", "lag_stats",
           "lag_destroy", "lag_last_error", "lag_nccl_unique_id", "lag_kernel_launches",
           "lag_abi_version", "lag_gridfill", "lag_ftle", "lag_stitch", "lag_local_group")


class LagError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class lag_config(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("global_nodes", ctypes.c_int64 * 3), ("origin", ctypes.c_double * 3),
                ("spacing", ctypes.c_double * 3), ("block_lo", ctypes.c_int64 * 3),
                ("block_hi", ctypes.c_int64 * 3), ("ghost", ctypes.c_int32),
                ("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("layout", ctypes.c_int32 * 3), ("exchange", ctypes.c_int32),
                ("row_pitch_bytes", ctypes.c_int64),
                ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


class lag_stats_t(ctypes.Structure):
    _fields_ = [("seeded", ctypes.c_int64), ("active", ctypes.c_int64),
                ("term_boundary", ctypes.c_int64), ("exit_domain", ctypes.c_int64),
                ("sent", ctypes.c_int64), ("received", ctypes.c_int64),
                ("particle_steps", ctypes.c_int64), ("cycles", ctypes.c_int64),
                ("device_error", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("phase_ms", ctypes.c_double * 3)]


_lib = None


def load(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"liblag.so not built at {path}: run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    lib.lag_init.argtypes = [P(lag_config), P(vp)]
    lib.lag_seed.argtypes = [vp, ctypes.c_int32, P(ctypes.c_int64)]
    lib.lag_advect_cycle.argtypes = [vp, vp, vp, ctypes.c_double]
    lib.lag_extract.argtypes = [vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int64, P(ctypes.c_int64),
                                ctypes.c_uint32]
    lib.lag_extract_ex.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int64, P(ctypes.c_int64),
                                   ctypes.c_uint32]
    lib.lag_local_group.argtypes = [P(vp), ctypes.c_int32]
    lib.lag_stats.argtypes = [vp, P(lag_stats_t)]
    lib.lag_destroy.argtypes = [vp]
    lib.lag_last_error.argtypes = [vp]
    lib.lag_last_error.restype = ctypes.c_char_p
    lib.lag_nccl_unique_id.argtypes = [vp, ctypes.c_int64]
    lib.lag_kernel_launches.argtypes = [vp]
    lib.lag_kernel_launches.restype = ctypes.c_int64
    lib.lag_abi_version.restype = ctypes.c_int32
    if lib.lag_abi_version() != LAG_ABI_VERSION:
        raise ImportError(f"{path} implements ABI {lib.lag_abi_version()}, the binding expects "
                          f"{LAG_ABI_VERSION}: rebuild with `python __graft_entry__.py build`")
    if hasattr(lib, "lag_stitch"):
        lib.lag_stitch.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_double), P(ctypes.c_double),
                                   ctypes.c_int32, vp, vp, ctypes.c_int64, vp, vp, vp, vp]
    if hasattr(lib, "lag_ftle"):
        lib.lag_ftle.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_double), ctypes.c_double,
                                 vp, vp, P(ctypes.c_int64), vp]
    if hasattr(lib, "lag_gridfill"):
        lib.lag_gridfill.argtypes = [ctypes.c_int32, P(ctypes.c_int64), ctypes.c_int32, vp, vp, vp, vp, vp]
    for name in ("lag_init", "lag_seed", "lag_advect_cycle", "lag_extract", "lag_extract_ex", "lag_stats",
                 "lag_destroy", "lag_nccl_unique_id", "lag_gridfill", "lag_ftle", "lag_stitch",
                 "lag_local_group"):
        if hasattr(lib, name):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _addr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):          # torch.Tensor
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if hasattr(x, "ctypes"):            # numpy array
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _check(st: int, ctx=None):
    if st != LAG_OK:
        msg = load().lag_last_error(ctx).decode(errors="replace")
        raise LagError(st, msg)


def lag_last_error(ctx=None) -> str:
    return load().lag_last_error(ctx).decode(errors="replace")


def lag_abi_version() -> int:
    return load().lag_abi_version()


def lag_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().lag_nccl_unique_id(buf, 128))
    return buf.raw


def make_config(dim: int, global_nodes: Sequence[int], origin: Sequence[float],
                spacing: Sequence[float], block_lo: Sequence[int], block_hi: Sequence[int],
                mode: int = LAG_BTO, ghost: int = 0, device: int = 0, rank: int = 0,
                nranks: int = 1, layout: Sequence[int] = (1, 1, 1),
                nccl_id: Optional[bytes] = None, stream: Optional[int] = None,
                exchange: int = 0, row_pitch_bytes: int = 0) -> lag_config:
    c = lag_config()
    c.dim, c.mode, c.ghost, c.device = dim, mode, ghost, device
    c.rank, c.nranks = rank, nranks
    c.exchange = int(exchange)
    c.row_pitch_bytes = int(row_pitch_bytes)
    for a in range(3):
        c.global_nodes[a] = int(global_nodes[a])
        c.origin[a] = float(origin[a])
        c.spacing[a] = float(spacing[a])
        c.block_lo[a] = int(block_lo[a])
        c.block_hi[a] = int(block_hi[a])
        c.layout[a] = int(layout[a])
    if nccl_id is not None:
        c._nccl_buf = ctypes.create_string_buffer(nccl_id, 128)   # keep alive with the struct
        c.nccl_id = ctypes.cast(c._nccl_buf, ctypes.c_void_p)
    c.stream = stream or None
    return c


def lag_init(cfg: lag_config) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    _check(load().lag_init(ctypes.byref(cfg), ctypes.byref(ctx)))
    return ctx


def lag_seed(ctx, stride: int) -> int:
    n = ctypes.c_int64(0)
    _check(load().lag_seed(ctx, int(stride), ctypes.byref(n)), ctx)
    return n.value


def lag_advect_cycle(ctx, v_t, v_t1, dt: float) -> None:
    _check(load().lag_advect_cycle(ctx, _addr(v_t), _addr(v_t1), float(dt)), ctx)


def lag_extract(ctx, interval_index: int, start=None, end=None, status=None,
                capacity: Optional[int] = None, flags: int = 0) -> int:
    """Returns n; outputs are written into the given buffers.  Latched async
    errors raise LagError after the outputs were written."""
    n = ctypes.c_int64(0)
    if capacity is None:
        caps = [x.shape[0] for x in (start, end, status) if x is not None]
        capacity = min(caps) if caps else 0
    _check(load().lag_extract(ctx, int(interval_index), _addr(start), _addr(end), _addr(status),
                              int(capacity), ctypes.byref(n), int(flags)), ctx)
    return n.value


def lag_extract_ex(ctx, interval_index: int, start=None, end=None, status=None, term_cycle=None,
                   capacity: Optional[int] = None, flags: int = 0) -> int:
    n = ctypes.c_int64(0)
    if capacity is None:
        caps = [x.shape[0] for x in (start, end, status, term_cycle) if x is not None]
        capacity = min(caps) if caps else 0
    _check(load().lag_extract_ex(ctx, int(interval_index), _addr(start), _addr(end), _addr(status),
                                 _addr(term_cycle), int(capacity), ctypes.byref(n), int(flags)), ctx)
    return n.value


def lag_local_group(ctxs) -> None:
    """Connect LAG_XCHG_LOCAL contexts (ctxs[r] = rank r) into one group."""
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value if isinstance(c, ctypes.c_void_p) else c for c in ctxs])
    _check(load().lag_local_group(arr, len(ctxs)))


def lag_stats(ctx) -> dict:
    s = lag_stats_t()
    _check(load().lag_stats(ctx, ctypes.byref(s)), ctx)
    d = {f: getattr(s, f) for f, _ in lag_stats_t._fields_ if f not in ("pad_", "phase_ms")}
    d["phase_ms"] = list(s.phase_ms)
    return d


def lag_destroy(ctx) -> None:
    _check(load().lag_destroy(ctx))


def lag_gridfill(values, valid, dims: Sequence[int], out=None, filled=None, stream=None):
    """GridFill reconstruction on a dense lattice (include/lag.h).  `values`
    [n, k] f64 and `valid` [n] u8 are device tensors in x-fastest lattice
    order; returns (out, filled), allocating them if not given."""
    import torch
    dim = len(dims)
    n = 1
    for d in dims:
        n *= int(d)
    k = values.shape[1]
    if out is None:
        out = torch.empty_like(values)
    if filled is None:
        filled = torch.empty_like(valid)
    if values.shape[0] != n or valid.shape[0] != n:
        raise ValueError("values/valid must hold prod(dims) nodes")
    d = (ctypes.c_int64 * 3)(*[int(x) for x in dims], *([1] * (3 - dim)))
    if stream is None:                  # (host tensors are rejected by the library)
        stream = torch.cuda.current_stream(values.device).cuda_stream if values.is_cuda else 0
    s = stream
    _check(load().lag_gridfill(dim, d, k, _addr(values), _addr(valid), _addr(out), _addr(filled), s))
    return out, filled


def lag_ftle(ends, dims: Sequence[int], spacing: Sequence[float], T: float, out=None, stream=None):
    """FTLE of a flow map on a dense lattice (include/lag.h).  `ends` [n, dim]
    f64 device tensor, x fastest.  Returns (ftle [n], n_degenerate)."""
    import torch
    dim = len(dims)
    if out is None:
        out = torch.empty((ends.shape[0],), dtype=torch.float64, device=ends.device)
    d = (ctypes.c_int64 * 3)(*[int(x) for x in dims], *([1] * (3 - dim)))
    sp = (ctypes.c_double * 3)(*[float(x) for x in spacing], *([1.0] * (3 - dim)))
    nd = ctypes.c_int64(0)
    if stream is None:
        stream = torch.cuda.current_stream(ends.device).cuda_stream if ends.is_cuda else 0
    _check(load().lag_ftle(dim, d, sp, float(T), _addr(ends), _addr(out), ctypes.byref(nd), stream))
    return out, nd.value


def lag_stitch(ends, starts, dims: Sequence[int], origin: Sequence[float], spacing: Sequence[float],
               valid=None, path=None, status=None, stream=None):
    """Stitch pathlines through K flow maps (include/lag.h).  `ends` [K, n, dim]
    f64 and `starts` [m, dim] f64 device tensors, `valid` [K, n] u8 or None.
    Returns (path [m, K+1, dim], status [m])."""
    import torch
    dim = len(dims)
    K, m = int(ends.shape[0]), int(starts.shape[0])
    if path is None:
        path = torch.empty((m, K + 1, dim), dtype=torch.float64, device=starts.device)
    if status is None:
        status = torch.empty((m,), dtype=torch.uint8, device=starts.device)
    d = (ctypes.c_int64 * 3)(*[int(x) for x in dims], *([1] * (3 - dim)))
    o = (ctypes.c_double * 3)(*[float(x) for x in origin[:dim]], *([0.0] * (3 - dim)))
    sp = (ctypes.c_double * 3)(*[float(x) for x in spacing[:dim]], *([1.0] * (3 - dim)))
    if stream is None:
        stream = torch.cuda.current_stream(starts.device).cuda_stream if starts.is_cuda else 0
    _check(load().lag_stitch(dim, d, o, sp, K, _addr(ends), _addr(valid), m, _addr(starts), _addr(path),
                             _addr(status), stream))
    return path, status


def lag_kernel_launches(ctx) -> int:
    return int(load().lag_kernel_launches(ctx))


class Context:
    """Owning handle for one block's lag_ctx (marshalling only)."""

    def __init__(self, cfg: lag_config):
        self.cfg = cfg
        self.dim = cfg.dim
        self.ctx = lag_init(cfg)
        self.n = 0
        self.interval = 0               # next lag_extract interval_index

    def seed(self, stride: int) -> int:
        self.n = lag_seed(self.ctx, stride)
        return self.n

    def advect(self, v_t, v_t1, dt: float) -> None:
        lag_advect_cycle(self.ctx, v_t, v_t1, dt)

    def extract(self, start=None, end=None, status=None, flags: int = 0, term_cycle=None) -> int:
        try:
            if term_cycle is not None:
                n = lag_extract_ex(self.ctx, self.interval, start, end, status, term_cycle, flags=flags)
            else:
                n = lag_extract(self.ctx, self.interval, start, end, status, flags=flags)
        except LagError as e:
            if e.status in LATCHED:          # outputs written, interval extracted, error reported
                self.interval += 1
            raise
        self.interval += 1
        return n

    def stats(self) -> dict:
        return lag_stats(self.ctx)

    def launches(self) -> int:
        return lag_kernel_launches(self.ctx)

    def close(self):
        if self.ctx is not None:
            lag_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """The blocks of a decomposition as LAG_XCHG_LOCAL COMM contexts on one
    device (marshalling only): cfgs[r] is rank r's configuration."""

    def __init__(self, cfgs):
        self.blocks = [Context(c) for c in cfgs]
        lag_local_group([b.ctx for b in self.blocks])

    def seed(self, stride: int):
        return [b.seed(stride) for b in self.blocks]

    def advect(self, v_t, v_t1, dt: float) -> None:
        """v_t[r], v_t1[r]: block r's device slices; the last call enqueues the cycle."""
        for b, a0, a1 in zip(self.blocks, v_t, v_t1):
            b.advect(a0, a1, dt)

    def extract(self, outs, flags: int = 0):
        """outs[r] = (start, end, status) device buffers of block r."""
        return [b.extract(*o, flags=flags) for b, o in zip(self.blocks, outs)]

    def stats(self):
        return [b.stats() for b in self.blocks]

    def close(self):
        for b in self.blocks:
            b.close()
