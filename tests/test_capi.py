"""CPU: the C-ABI library loads, exports every entry point declared in
include/*.h, and the product path fails loudly (no CPU fallback) when no
CUDA device is present."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        txt = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(lrcvt_\w+)\s*\(", txt))
    return sorted(names)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("lrcvt_plan_create", "lrcvt_classify", "lrcvt_centroidal_update", "lrcvt_isobands",
                 "lrcvt_label_components", "lrcvt_aggregate", "lrcvt_segment_hit_t"):
        assert must in syms


def test_library_exports_all_declared_symbols():
    from paper_2208_06970_b200 import _lib

    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert L.lrcvt_version() >= 1


def test_ctypes_signatures_cover_header():
    from paper_2208_06970_b200 import _lib

    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def declared_arities():
    out = {}
    for h in (ROOT / "include").glob("*.h"):
        txt = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for name, params in re.findall(r"\b(lrcvt_\w+)\s*\(([^)]*)\)\s*;", txt):
            params = params.strip()
            out[name] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_ctypes_arity_matches_header():
    """A ctypes argtypes list shorter than the C prototype silently passes the
    trailing arguments as C int (a truncated stream pointer crashes)."""
    from paper_2208_06970_b200 import _lib

    for name, arity in declared_arities().items():
        if name in _lib.SIGNATURES:
            assert len(_lib.SIGNATURES[name][1]) == arity, name


def test_bad_arguments_rejected_without_device():
    """Argument validation happens before any device work."""
    from paper_2208_06970_b200 import _lib

    L = _lib.lib()
    rc = L.lrcvt_isobands(10, None, None, 1, None, None)
    assert rc == -2
    assert b"bad arguments" in L.lrcvt_last_error()


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2208_06970_b200 import IsobandSpec, VoxelGrid, classify_isobands
    from paper_2208_06970_b200._lib import LrcvtCudaError

    g = VoxelGrid((4, 1, 1), (1, 1, 1), {"f": np.zeros(4, np.float32)})
    with pytest.raises(LrcvtCudaError):
        classify_isobands(g, IsobandSpec("f", [0.0, 1.0]))


def test_new_entry_points_validate_arguments_without_device():
    """§8(f) entry points reject bad arguments before touching the device."""
    import ctypes

    from paper_2208_06970_b200 import _lib

    L = _lib.lib()
    n_in, n_runs, tot = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    rc = L.lrcvt_seed_masses(4, 4, 4, 2, None, 1, 0, None, 10, 10, None, None, None, None, None, None,
                             ctypes.byref(n_in), ctypes.byref(n_runs), ctypes.byref(tot), None)
    assert rc == -2 and b"lrcvt_seed_masses" in L.lrcvt_last_error()
    got = ctypes.c_int64()
    rc = L.lrcvt_layout_records(4, 4, 4, 1, None, None, None, 1, 1, 10, None, None, None, None, ctypes.byref(got),
                                None)
    assert rc == -2 and b"lrcvt_layout_records" in L.lrcvt_last_error()
    rc = L.lrcvt_region_adjacency(4, 4, 4, None, None, 3, 10, None, ctypes.byref(got), None)
    assert rc == -2 and b"lrcvt_region_adjacency" in L.lrcvt_last_error()


@pytest.mark.parametrize("n_inband", [0, 1, 2047, 2048, 2049, 5_000_000, (1 << 29) - 1, 1 << 29, (1 << 29) + 1,
                                      (1 << 30) + 12345, (1 << 31) - 2])
def test_round_classes_cover_inband_without_overflow(n_inband):
    """Size classes of the round graph (lrcvt_capi.cu build_round_graph): every
    class launches between 1 and n_inband voxels (< 2^31, so the int launch
    arithmetic cannot wrap -- the class cap 2^31 above 2^29 in-band voxels
    did), the launch sizes grow, and the last class covers the whole in-band
    set (a sweep or phase-2 start evaluates all of it)."""
    import ctypes

    from paper_2208_06970_b200 import _lib

    L = _lib.lib()
    buf = (ctypes.c_int64 * 16)()
    n = L.lrcvt_round_classes(n_inband, buf, 16)
    assert 1 <= n <= 12
    items = [buf[i] for i in range(n)]
    nin = max(n_inband, 1)
    assert all(1 <= it <= nin < 2**31 for it in items)
    assert items == sorted(items)
    assert items[-1] == nin
    # the eval launch grid of the largest class fits an int
    assert (items[-1] + 63) // 64 < 2**31
    assert L.lrcvt_round_classes(-1, buf, 16) < 0
