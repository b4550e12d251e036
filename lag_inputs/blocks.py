"""Uniform grid + simulation-owned domain decomposition (input plumbing).

The paper takes the decomposition as given by the simulation (PAPER.md:135,
§2.2 "domain decomposition and distribution are simulation-determined").  We
follow SPEC.md:98-106 (domain/decompose) for the near-equal split with the
remainder spread to low-index blocks, and SURVEY.md §8(b) for the slice
extent: per axis ``(min(hi+1, N) - lo) + 2G`` nodes.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class Grid:
    dim: int                      # 2 or 3
    nodes: Tuple[int, int, int]   # N_a (unused axis = 1)
    origin: Tuple[float, float, float]
    spacing: Tuple[float, float, float]

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")

    @property
    def extent(self):
        return tuple((self.nodes[a] - 1) * self.spacing[a] for a in range(self.dim))


@dataclasses.dataclass(frozen=True)
class Block:
    rank: int
    coords: Tuple[int, int, int]   # block coordinates in the layout
    lo: Tuple[int, int, int]       # owned node range [lo, hi) per axis
    hi: Tuple[int, int, int]


def _split(n: int, parts: int) -> List[int]:
    """Cut points of ``n`` nodes into ``parts`` near-equal ranges (remainder to
    low-index blocks: 10 nodes over 3 -> 4/3/3)."""
    if parts < 1 or parts > n:
        raise ValueError(f"cannot split {n} nodes into {parts} blocks")
    base, rem = divmod(n, parts)
    cuts = [0]
    for p in range(parts):
        cuts.append(cuts[-1] + base + (1 if p < rem else 0))
    return cuts


def decompose(grid: Grid, layout: Sequence[int]) -> List[Block]:
    """Blocks in x-fastest rank order (rank = bx + Lx*(by + Ly*bz))."""
    lay = tuple(layout) + (1,) * (3 - len(layout))
    cuts = [_split(grid.nodes[a], lay[a]) if a < grid.dim else [0, 1] for a in range(3)]
    blocks = []
    for bz in range(lay[2]):
        for by in range(lay[1]):
            for bx in range(lay[0]):
                c = (bx, by, bz)
                lo = tuple(cuts[a][c[a]] for a in range(3))
                hi = tuple(cuts[a][c[a] + 1] for a in range(3))
                rank = bx + lay[0] * (by + lay[1] * bz)
                blocks.append(Block(rank, c, lo, hi))
    return blocks


def layout_for(nranks: int, dim: int = 3) -> Tuple[int, int, int]:
    """(1,1,1), (2,1,1), (2,2,1), (2,2,2), ... : double the smallest axis."""
    lay = [1, 1, 1]
    n = nranks
    a = 0
    while n > 1:
        if n % 2:
            raise ValueError("rank count must be a power of two")
        lay[a % dim] *= 2
        n //= 2
        a += 1
    return tuple(lay)


def block_slice_extent(grid: Grid, block: Block, ghost: int) -> Tuple[int, int, int]:
    """Nodes per axis of a block's slice array (SURVEY.md §8(b) lag_config)."""
    ext = []
    for a in range(3):
        if a >= grid.dim:
            ext.append(1)
            continue
        n = min(block.hi[a] + 1, grid.nodes[a]) - block.lo[a] + 2 * ghost
        ext.append(n)
    return tuple(ext)


def cut_block_slice(global_nodes, grid: Grid, block: Block, ghost: int):
    """Copy a block's slice (owned + shared upper plane + G ghost layers) out of
    a global node array shaped [Nz, Ny, Nx, dim] (x fastest).  Ghost nodes that
    fall outside the global grid are zero (allocated, never read).  Works for
    numpy arrays and torch tensors."""
    ext = block_slice_extent(grid, block, ghost)
    is_np = isinstance(global_nodes, np.ndarray)
    if is_np:
        out = np.zeros((ext[2], ext[1], ext[0], grid.dim), dtype=global_nodes.dtype)
    else:
        import torch
        out = torch.zeros((ext[2], ext[1], ext[0], grid.dim), dtype=global_nodes.dtype,
                          device=global_nodes.device)
    src, dst = [], []
    for a in range(3):
        if a >= grid.dim:
            src.append(slice(0, 1)); dst.append(slice(0, 1)); continue
        g0 = block.lo[a] - ghost
        g1 = g0 + ext[a]
        s0, s1 = max(g0, 0), min(g1, grid.nodes[a])
        src.append(slice(s0, s1)); dst.append(slice(s0 - g0, s1 - g0))
    out[dst[2], dst[1], dst[0]] = global_nodes[src[2], src[1], src[0]]
    return out


def seed_lattice_count(lo: int, hi: int, stride: int) -> int:
    """Number of lattice nodes g = k*stride with lo <= g < hi (input bookkeeping
    used to size caller buffers)."""
    return -(-hi // stride) - (-(-lo // stride))
