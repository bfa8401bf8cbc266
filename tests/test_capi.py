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
