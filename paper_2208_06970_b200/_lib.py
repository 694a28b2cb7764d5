"""ctypes binding of the C-ABI library ``liblrcvt_cuda.so`` (include/lrcvt_cuda.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2208_06970_b200/csrc``). There is no CPU fallback: every
entry point of this package fails loudly when the library or a CUDA device is
missing.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

import os

# LRCVT_LIB overrides the in-tree library (A/B timing of two builds)
LIB_PATH = Path(os.environ.get("LRCVT_LIB") or Path(__file__).resolve().with_name("liblrcvt_cuda.so"))

W_ONES, W_F64, W_F32_G1, W_F32_G2 = 0, 1, 2, 3
E_CUDA, E_ARG, E_NOMEM = -1, -2, -3


class ClassifyStats(ctypes.Structure):
    _fields_ = [
        ("rounds", c_int64),
        ("sweeps", c_int64),
        ("assigned", c_int64),
        ("evaluations", c_int64),
        ("commits", c_int64),
        ("bad_sites", c_int64),
        ("phase1_rounds", c_int64),
        ("eligible", c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


# name -> (restype, argtypes); mirrors include/lrcvt_cuda.h exactly
SIGNATURES = {
    "lrcvt_version": (c_int, []),
    "lrcvt_last_error": (ctypes.c_char_p, []),
    "lrcvt_plan_create": (
        c_int,
        [POINTER(c_void_p), c_int64, c_int64, c_int64, c_double, c_double, c_double,
         c_void_p, c_int32, c_int64, c_void_p],
    ),
    "lrcvt_plan_destroy": (c_int, [c_void_p]),
    "lrcvt_plan_inband": (c_int64, [c_void_p]),
    "lrcvt_classify": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(ClassifyStats), c_void_p],
    ),
    "lrcvt_centroidal_update": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_double,
         c_void_p, c_void_p, c_void_p, POINTER(c_int64), c_void_p],
    ),
    "lrcvt_plan_reuse_eligible": (c_int, [c_void_p, c_int]),
    "lrcvt_unpack_site_src": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "lrcvt_segment_hit_t": (
        c_int,
        [c_int64, c_int64, c_int64, c_double, c_double, c_double, c_void_p, c_void_p,
         c_void_p, c_int64, c_void_p, c_void_p],
    ),
    "lrcvt_segment_clear_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "lrcvt_plan_set_timing": (c_int, [c_void_p, c_int]),
    "lrcvt_plan_timing": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_double)]),
    "lrcvt_launch_count": (ctypes.c_ulonglong, []),
    "lrcvt_plan_profile": (c_int, [c_void_p, POINTER(c_double)]),
    "lrcvt_round_classes": (c_int32, [c_int64, POINTER(c_int64), c_int32]),
    "lrcvt_mg_set_slab": (c_int, [c_void_p, c_int64, c_int64]),
    "lrcvt_mg_state": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "lrcvt_mg_set_peers": (c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "lrcvt_mg_begin": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int64),
                               c_void_p]),
    "lrcvt_mg_phase2": (c_int, [c_void_p, c_int64, c_void_p, POINTER(c_int64), c_void_p]),
    "lrcvt_mg_eval": (c_int, [c_void_p, c_int32, c_int32, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
                              c_void_p]),
    "lrcvt_mg_boundary": (c_void_p, [c_void_p, c_int32]),
    "lrcvt_mg_commit": (c_int, [c_void_p, c_void_p, c_int64, c_int32, POINTER(c_int64), POINTER(c_int64), c_void_p]),
    "lrcvt_mg_finish": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_int64), c_void_p]),
    "lrcvt_mg_vote_exact": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "lrcvt_mg_vote_exact_finish": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "lrcvt_mg_vote_box": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "lrcvt_mg_vote_scan": (c_int, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int32, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    "lrcvt_mg_vote_carry": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrcvt_mg_move": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_void_p,
                              POINTER(c_int64), c_void_p]),
    "lrcvt_mg_timing": (c_int, [c_void_p, c_int32, POINTER(c_double)]),
    "lrcvt_ipc_export": (c_int, [c_void_p, c_void_p]),
    "lrcvt_ipc_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "lrcvt_ipc_close": (c_int, [c_void_p]),
    "lrcvt_plan_persistent_outputs": (c_int, [c_void_p, c_int]),
    "lrcvt_isobands": (
        c_int,
        [c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_void_p],
    ),
    "lrcvt_label_components": (
        c_int,
        [c_int64, c_int64, c_int64, c_void_p, c_int32, c_void_p, POINTER(c_int32), c_void_p],
    ),
    "lrcvt_component_table": (
        c_int,
        [c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p,
         c_void_p],
    ),
    "lrcvt_aggregate": (
        c_int,
        [c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p,
         c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "lrcvt_seed_masses": (
        c_int,
        [c_int64, c_int64, c_int64, c_int32, c_void_p, c_int32, c_int32, c_void_p, c_int64, c_int64,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int64), POINTER(c_int64),
         POINTER(c_double), c_void_p],
    ),
    "lrcvt_layout_records": (
        c_int,
        [c_int64, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p, POINTER(c_int64), c_void_p],
    ),
    "lrcvt_region_adjacency": (
        c_int,
        [c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_void_p, POINTER(c_int64), c_void_p],
    ),
}

_lib = None


class LrcvtCudaError(RuntimeError):
    pass


def lib():
    """Load the library once; raise if it is absent (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LrcvtCudaError(
            f"CUDA extension missing: {LIB_PATH} not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    L = lib()
    return [name for name in SIGNATURES if hasattr(L, name)]


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = lib().lrcvt_last_error().decode(errors="replace")
        raise LrcvtCudaError(f"{what} failed ({rc}): {msg}")
    return rc


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise LrcvtCudaError("no CUDA device: the LSRCVT hot path runs only on the GPU")
    lib()
    return torch


def stream_handle(torch) -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
