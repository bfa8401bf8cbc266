"""CPU-only checks of the drop-in boundary: libsk200.so loads (no GPU needed)
and exports exactly the entry points include/sk200.h declares."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sk200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(sk_\w+)\s*\(", src, re.M)))


def test_header_parses():
    names = declared()
    assert "sk_conv_forward" in names and "sk_kmap_build" in names
    assert len(names) >= 25


def test_library_loads_and_exports_every_symbol():
    from paper_2311_12862_b200 import _lib
    L = _lib.lib()
    for name in declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (sk_\w+)", out))
    assert exported == set(declared())
    assert set(_lib.SYMBOLS) == set(declared())


def test_version_and_error_without_gpu():
    from paper_2311_12862_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.sk_version()
    # no device here: creating a context must fail loudly, not fall back
    p = ctypes.c_void_p()
    rc = L.sk_ctx_create(0, ctypes.byref(p))
    import torch
    if not torch.cuda.is_available():
        assert rc == 3  # SK_ERR_CUDA
        assert L.sk_last_error()


def test_cubin_is_sm100a_with_tcgen05():
    from paper_2311_12862_b200 import _lib
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCMMA" in out  # tcgen05.mma
    assert "LDTM" in out                           # tcgen05.ld


def test_tuner_space_without_gpu():
    """default_space (tuner.cpp:9-26) is host code: the reference's 12 configs
    in its order, then the B200 kernel variants the TilePreset fields select
    (one CTA per SM, TMA gather4, 32-channel stages, one-tile work items)."""
    from paper_2311_12862_b200.network import default_space
    from paper_2311_12862_b200 import sparse as sk
    space = default_space()
    ref = [sk.DataflowConfig(sk.GATHER_GEMM_SCATTER), sk.DataflowConfig(sk.FETCH_ON_DEMAND)]
    for s in range(5):
        for t in (sk.tile_small(), sk.tile_large()):
            ref.append(sk.DataflowConfig(sk.IMPLICIT_GEMM, s, t))
    assert space[:12] == ref
    extra = space[12:]
    assert len(extra) == 9 and all(c.kind == sk.IMPLICIT_GEMM for c in extra)
    assert {c.tile.cta_m for c in extra} == {64, 128, 256}
    assert any(c.tile.load_width == 1 for c in extra)      # TMA gather4
    assert any(c.tile.cta_k == 32 for c in extra)          # single-slab 32-channel stages
    assert len({c.name() for c in space}) == len(space)    # names tell the variants apart
