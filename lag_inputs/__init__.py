"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no RK4, no interpolation, no
boundary tests).  It only produces:

* velocity slices: analytic fields evaluated at grid nodes in fp64 and rounded
  once to fp32 (``fields``), laid out AoS (x, y[, z]) per node, x fastest;
* block geometry: the simulation-owned domain decomposition (``blocks``) and
  cutting a block's slice (owned nodes + shared upper plane + ghost layers)
  out of a global node array.

Both ``oracle/`` and the product tests/bench import it; neither side imports
the other.  Recipes are documented in DESIGN.md §"Input recipe".
"""
from .blocks import Grid, Block, decompose, block_slice_extent, cut_block_slice, layout_for
from .fields import (FieldSpec, make_config, field_at_nodes, config_names,
                     CONFIGS)

__all__ = ["Grid", "Block", "decompose", "block_slice_extent", "cut_block_slice",
           "layout_for", "FieldSpec", "make_config", "field_at_nodes",
           "config_names", "CONFIGS"]
