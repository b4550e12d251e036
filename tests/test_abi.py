"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/lag.h declares, validates configurations, and fails loudly
(no CPU fallback) when no GPU is present.  No compute call runs here."""
import os
import re
import subprocess

import pytest

import paper_2004_02003_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "lag.h")).read()
    return sorted(set(re.findall(r"LAG_API\s+[\w\s\*]+?\b(lag_\w+)\s*\(", src)))


def test_header_declares_the_binding_exports():
    assert declared_functions() == sorted(P.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = P.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lag_\w+)", out))
    assert set(declared_functions()) <= exported
    assert P.lag_abi_version() == P.LAG_ABI_VERSION == 3


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kw,frag", [
    (dict(dim=4), "dim"),
    (dict(global_nodes=(1, 8, 8)), "global_nodes"),
    (dict(block_hi=(9, 8, 8)), "block"),
    (dict(block_lo=(4, 0, 0), block_hi=(4, 8, 8)), "block"),
    (dict(spacing=(0.0, 1.0, 1.0)), "spacing"),
    (dict(spacing=(float("nan"), 1.0, 1.0)), "spacing"),
    (dict(origin=(float("inf"), 0.0, 0.0)), "origin"),
    (dict(mode=7), "mode"),
    (dict(mode=1, ghost=0, nranks=2, layout=(2, 1, 1), nccl_id=b"x" * 128), "ghost"),
    (dict(ghost=-1), "ghost"),
    (dict(mode=1, ghost=1, nranks=2, layout=(2, 1, 1)), "nccl_id"),
    (dict(mode=1, ghost=1, nranks=2, layout=(3, 1, 1)), "layout"),
    (dict(global_nodes=(2 ** 12, 2 ** 12, 2 ** 12), block_hi=(2 ** 12, 2 ** 12, 2 ** 12)), "bits"),
    (dict(row_pitch_bytes=12 * 7), "row_pitch"),          # shorter than a row of 8 nodes
    (dict(row_pitch_bytes=100), "row_pitch"),             # not whole nodes
    (dict(mode=1, ghost=1, nranks=65, layout=(65, 1, 1), global_nodes=(130, 8, 8), block_hi=(2, 8, 8),
          exchange=3), "64"),
])
def test_init_rejects_bad_configurations(kw, frag):
    base = dict(dim=3, global_nodes=(8, 8, 8), origin=(0, 0, 0), spacing=(1, 1, 1),
                block_lo=(0, 0, 0), block_hi=(8, 8, 8))
    base.update(kw)
    cfg = P.make_config(**base)
    with pytest.raises(P.LagError) as e:
        P.lag_init(cfg)
    assert e.value.status == P.LAG_EINVAL
    assert frag.split()[0] in str(e.value) or "too large" in str(e.value)


def test_unused_axis_must_be_trivial_in_2d():
    cfg = P.make_config(2, (8, 8, 2), (0, 0, 0), (1, 1, 1), (0, 0, 0), (8, 8, 2))
    with pytest.raises(P.LagError) as e:
        P.lag_init(cfg)
    assert e.value.status == P.LAG_EINVAL


def test_valid_config_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = P.make_config(3, (8, 8, 8), (0, 0, 0), (1, 1, 1), (0, 0, 0), (8, 8, 8))
    with pytest.raises(P.LagError) as e:
        P.lag_init(cfg)
    assert e.value.status == P.LAG_ECUDA


def test_null_context_calls_are_rejected():
    with pytest.raises(P.LagError):
        P.lag_seed(None, 1)
    with pytest.raises(P.LagError):
        P.lag_advect_cycle(None, 1, 1, 0.1)
    assert "NULL" in P.lag_last_error(None) or P.lag_last_error(None)


def test_product_never_imports_the_oracle():
    """The product path shares no code with oracle/ (DESIGN.md §boundary)."""
    pkg = os.path.join(ROOT, "paper_2004_02003_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                txt = open(path).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), path
            elif f.endswith((".cu", ".cuh", ".h", ".cpp")):
                txt = open(path).read()
                assert "lag_oracle" not in txt and "orc_" not in txt, path


def test_gridfill_rejects_null_and_bad_sizes_without_a_gpu():
    import ctypes
    lib = P.load()
    dims = (ctypes.c_int64 * 3)(4, 4, 1)
    assert lib.lag_gridfill(2, dims, 2, None, None, None, None, None) == P.LAG_EINVAL
    assert lib.lag_gridfill(4, dims, 2, 1, 1, 1, 1, None) == P.LAG_EINVAL
    assert lib.lag_gridfill(2, dims, 0, 1, 1, 1, 1, None) == P.LAG_EINVAL
    assert "gridfill" in P.lag_last_error(None)


def test_ftle_rejects_bad_arguments_without_a_gpu():
    import ctypes
    lib = P.load()
    dims = (ctypes.c_int64 * 3)(4, 4, 4)
    sp = (ctypes.c_double * 3)(1.0, 1.0, 1.0)
    assert lib.lag_ftle(3, dims, sp, 1.0, None, None, None, None) == P.LAG_EINVAL
    assert lib.lag_ftle(3, dims, sp, 0.0, 1, 1, None, None) == P.LAG_EINVAL
    assert lib.lag_ftle(1, dims, sp, 1.0, 1, 1, None, None) == P.LAG_EINVAL
    bad = (ctypes.c_double * 3)(1.0, -1.0, 1.0)
    assert lib.lag_ftle(3, dims, bad, 1.0, 1, 1, None, None) == P.LAG_EINVAL


def test_stitch_rejects_bad_arguments_without_a_gpu():
    import ctypes
    lib = P.load()
    dims = (ctypes.c_int64 * 3)(4, 4, 4)
    o = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
    sp = (ctypes.c_double * 3)(1.0, 1.0, 1.0)
    assert lib.lag_stitch(3, dims, o, sp, 1, None, None, 5, 1, 1, 1, None) == P.LAG_EINVAL   # ends NULL
    assert lib.lag_stitch(3, dims, o, sp, -1, 1, None, 5, 1, 1, 1, None) == P.LAG_EINVAL
    one = (ctypes.c_int64 * 3)(4, 1, 4)
    assert lib.lag_stitch(3, one, o, sp, 1, 1, None, 5, 1, 1, 1, None) == P.LAG_EINVAL    # extent < 2
    assert lib.lag_stitch(3, dims, o, sp, 1, 1, None, 0, None, None, None, None) == P.LAG_OK  # no pathlines
