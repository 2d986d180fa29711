"""The C-ABI library loads without a GPU and exports exactly what include/*.h declares."""
import glob
import os
import re
import subprocess

import pytest

from paper_2403_13135_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"^\s*int\s+(ice_\w+)\s*\(", src, flags=re.M))
    return names


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T ice_" in line}


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2403_13135_b200.csrc import build
        build.build()


def test_library_loads_and_binds():
    lib = _native.load()
    for name in _native.SIGNATURES:
        assert getattr(lib, name).restype is not None


def test_every_declared_symbol_is_exported_and_bound():
    decl = declared()
    assert decl, "no entry points parsed from include/*.h"
    assert decl <= exported()
    assert decl == set(_native.SIGNATURES), decl ^ set(_native.SIGNATURES)


def test_argument_errors_are_reported_before_launch():
    lib = _native.load()
    cfg = _native.IceFilterCfg(7, 21, 3, 0, 128, 0, 16)
    sc = _native.IceScheme()
    # n < 0 and a window larger than the tile are rejected host-side (no device needed)
    assert lib.ice_autolabel(None, -1, 16, 16, cfg, sc, None, None, None, None, None, None, None) == -1
    assert lib.ice_autolabel(1, 1, 16, 16, cfg, sc, 1, 1, None, 1, 1, 1, None) == -2
    assert lib.ice_autolabel(1, 1, 300, 300, cfg, sc, 1, 1, None, 1, 1, 1, None) == -3


def test_autolabel_scene_scratch_query_and_errors():
    """ice_autolabel_scene (region path beyond 256 x 256): CUB-style scratch query and the
    host-side argument checks, all before any device work."""
    import ctypes
    lib = _native.load()
    cfg = _native.IceFilterCfg(7, 21, 3, 0, 128, 0, 16)
    sc = _native.IceScheme()
    q = ctypes.c_uint64(123)
    args = (None, None, None, None, None, None)
    assert lib.ice_autolabel_scene(None, 2, 512, 512, cfg, sc, *args, None, ctypes.byref(q), None) == 0
    assert q.value == ((2 * 4152 + 255) // 256) * 256 + 2 * (2 * 512 * 512)  # SWAR windows: d + bg planes
    assert lib.ice_autolabel_scene(None, 2, 512, 520, cfg, sc, *args, None, ctypes.byref(q), None) == 0
    assert q.value == ((2 * 4152 + 255) // 256) * 256 + ((2 * 512 * 520 + 255) // 256) * 256  # generic: d plane
    assert lib.ice_autolabel_scene(None, 3, 64, 64, cfg, sc, *args, None, ctypes.byref(q), None) == 0
    assert q.value == 0  # <= 256 x 256: one CTA per tile, no scratch
    assert lib.ice_autolabel_scene(None, 1, 300, 10, cfg, sc, *args, None, ctypes.byref(q), None) == -2
    small = ctypes.c_uint64(1000)
    assert lib.ice_autolabel_scene(1, 1, 600, 600, cfg, sc, 1, 1, None, 1, 1, 1, 1, ctypes.byref(small), None) == -5
    big = _native.IceFilterCfg(7, 241, 3, 0, 128, 0, 16)  # halo 123: cores would be < 16 px
    assert lib.ice_autolabel_scene(None, 1, 600, 600, big, sc, *args, None, ctypes.byref(q), None) == -3
    assert lib.ice_autolabel_set_path(4) == -1
