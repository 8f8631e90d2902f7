"""CPU checks of the C-ABI boundary: the library builds, loads, and exports every
symbol include/nemdcell.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from paper_1412_3784_b200 import build as B
from paper_1412_3784_b200 import nemdcell

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "nemdcell.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nc_[a-z_]+)\s*\(", txt)))


def test_library_builds_and_exports_every_header_symbol():
    B.build()
    lib = ctypes.CDLL(B.LIB)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(nemdcell.EXPORTS) == syms


def test_version_and_create_error_paths_without_gpu():
    lib = nemdcell.load()
    assert b"sm_100a" in lib.nc_version()
    # invalid configuration is rejected before any device work
    cfg = nemdcell.nc_config()
    cfg.variant = 7
    h = ctypes.c_void_p()
    st = lib.nc_create(ctypes.byref(cfg), ctypes.byref(h))
    assert st == 1 and not h.value
    assert b"variant" in lib.nc_last_error(None)


def test_sass_is_sm100a():
    """The shipped library holds sm_100a SASS for every kernel of the path."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-symbols", B.LIB], capture_output=True, text=True).stdout
    for k in ("k_pairs", "k_wrap_key", "k_rank_gather", "k_kick_drift_key", "k_scan_apply"):
        assert k in out, k
