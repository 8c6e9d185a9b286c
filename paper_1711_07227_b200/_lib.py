"""ctypes binding of liblcrwmd.so (include/lcrwmd.h).

This is the whole boundary between the Python mirror of the reference API and
the CUDA kernels: plain pointers, sizes and a cudaStream_t, status codes
mapped back to the reference's exception types (ValueError for bad
arguments, RuntimeError for CUDA failures).  There is no fallback: if the
library or a CUDA device is missing, every call raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("LCRW_LIB", Path(__file__).resolve().parent / "liblcrwmd.so"))

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
SZ = C.c_size_t

# name -> (restype, argtypes); mirrors include/lcrwmd.h
SIGNATURES: dict[str, tuple] = {
    "lcrw_abi_version": (I32, []),
    "lcrw_status_string": (C.c_char_p, [I32]),
    "lcrw_last_error": (C.c_char_p, []),
    "lcrw_sm_count": (I32, [P]),
    "lcrw_padded_dim": (I32, [I32]),
    "lcrw_operand_k": (I32, [I32, I32]),
    "lcrw_max_sqnorm": (I32, [P, I64, I32, P, P]),
    "lcrw_scale_from_max_sqnorm": (I32, [P, P, P]),
    "lcrw_prepare_rows": (I32, [P, I64, I32, I32, I32, P, P, P, P]),
    "lcrw_gather_rows": (I32, [P, P, I32, P, I64, P, P, P]),
    "lcrw_row_classes_workspace": (I32, [I64, P]),
    "lcrw_row_classes": (I32, [P, I64, I32, P, P, P, P, P, P, SZ, P]),
    "lcrw_match_rows": (I32, [P, I64, P, I32, P, P, I64, P, P, P]),
    "lcrw_restrict_workspace": (I32, [I64, P]),
    "lcrw_restrict": (I32, [P, I64, I64, P, P, P, P, SZ, P]),
    "lcrw_remap_ids": (I32, [P, I64, P, P, P]),
    "lcrw_endmask_words": (I64, [I64]),
    "lcrw_plan_ranges": (I64, [I64, I32]),
    "lcrw_segment_plan": (I32, [P, I64, I64, I64, I32, P, P, I64, P]),
    "lcrw_phase1": (I32, [P, P, I64, P, I64, I32, I32, P, I64, I64, P, P, I64, P, P, I64, I32, P]),
    "lcrw_zero_identical": (I32, [P, I64, P, P, P, P, I64, I32, P]),
    "lcrw_spmm": (I32, [P, P, P, I64, P, I64, I32, I64, I64, I64, P, I64, I64, P]),
    "lcrw_spmm_dist": (I32, [P, P, P, I64, P, I64, I32, I64, I64, I64, P, I64, I64, P]),
    "lcrw_reverse_workspace": (I32, [I64, I32, I64, I64, P]),
    "lcrw_reverse_pipeline": (I32, [P, P, I64, P, I64, I32, I32, P, P, P, I64, P, P, P, P, P, P, I64, P, I64, P, I64,
                                    I64, P, P, I32, I64, I64, I32, P, P, I64, I32, P, I32, P, P, P, SZ, P]),
    "lcrw_table_chunk": (I32, []),
    "lcrw_table_bytes": (I64, [I64, I64]),
    "lcrw_table_operand_rows": (I64, [I64]),
    "lcrw_table_transpose": (I32, [P, P, I64, I64, P, P, P]),
    "lcrw_distance_table": (I32, [P, P, I64, P, I64, I32, I32, P, P, P, I64, P, P, P, P, P, P]),
    "lcrw_table_min": (I32, [P, I64, I64, P, I64, I64, P, P, P, I64, P, P, P, I64, P]),
    "lcrw_refine_tau": (C.c_float, []),
    "lcrw_refine_near": (I32, [P, I64, I32, I64, I64, P, I64, P, P, P, P, I32, P, P, P, P, I64, I32, P]),
    "lcrw_near_pairs_workspace": (I32, [I64, I64, I64, P]),
    "lcrw_near_pairs_build": (I32, [P, I64, I64, P, P, P, P, I32, P, P, I64, P, P]),
    "lcrw_near_pairs_reset": (I32, [I64, I64, I64, P, P]),
    "lcrw_near_pairs_candidates": (I32, [P, I64, I64, I64, I64, P, P, I32, P, I64, P, P]),
    "lcrw_near_pairs_finish": (I32, [I64, I64, P, P, P, P, I32, P, I64, P, P]),
    "lcrw_near_scatter": (I32, [P, I64, I64, I64, I32, P, I64, I32, I64, P, I64, P, P, P, P, P]),
    "lcrw_symmetrize_max": (I32, [P, I64, I64, P]),
    "lcrw_max_transposed": (I32, [P, I64, P, I64, I64, I64, P]),
    "lcrw_max_transposed_into": (I32, [P, I64, P, I64, P, I64, I64, I64, P]),
    "lcrw_reverse_panels_tile_rows": (I32, []),
    "lcrw_reverse_panels_group": (I32, []),
    "lcrw_reverse_panels_warps": (I32, []),
    "lcrw_reverse_panels_ilp": (I32, []),
    "lcrw_reverse_panels": (I32, [P, I64, I64, I64, I64, P, P, I64, P, I64, P, I64, I64, P, P, I32, I64, P]),
    "lcrw_reverse_panels_top_slots": (I32, []),
    "lcrw_plan_reverse_words_bound": (I64, [I64, I64, I64, I32, I32, I32, I32]),
    "lcrw_plan_reverse": (I32, [P, I64, P, P, P, I64, I32, I32, I32, I32, P, I64, P, P]),
    "lcrw_topk_rows_workspace": (I32, [I64, I64, I32, P]),
    "lcrw_emd_problem_bytes": (SZ, [I32, I32]),
    "lcrw_emd_batch": (I32, [P, P, P, P, P, P, P, I64, I32, P, P, I64, I32, I32, P, P, P, P, P]),
    "lcrw_topk_rows": (I32, [P, I64, I64, I64, I64, I32, P, P, P, SZ, P]),
    "lcrw_profile_reset": (I32, [I32]),
    "lcrw_profile_count": (I64, []),
    "lcrw_profile_get": (I32, [I64, C.c_char_p, I32, P]),
    "lcrw_topk_segments": (I32, [P, P, I64, I64, I32, P, P, P]),
    "lcrw_topk_sort_workspace": (I32, [I64, P]),
    "lcrw_topk_sort": (I32, [P, P, I64, I64, P, P, P, SZ, P]),
    "lcrw_topk_sort_any_workspace": (I32, [I64, P]),
    "lcrw_squared_norms": (I32, [P, I32, I64, I64, P, P]),
    "lcrw_euclidean_f64": (I32, [P, P, I64, P, P, I64, I64, P, I32, I64, P]),
    "lcrw_segmented_min": (I32, [P, I32, I64, I64, I64, P, I64, P, P]),
    "lcrw_topk_sort_any": (I32, [P, I32, P, I64, I64, P, P, P, SZ, P]),
}

# functions returning a value rather than a status
_VALUE_FUNCS = {"lcrw_emd_problem_bytes", "lcrw_abi_version", "lcrw_status_string", "lcrw_last_error", "lcrw_padded_dim", "lcrw_operand_k",
                "lcrw_endmask_words", "lcrw_plan_ranges", 
                "lcrw_reverse_panels_tile_rows", "lcrw_reverse_panels_group", "lcrw_reverse_panels_warps",
                "lcrw_reverse_panels_ilp", "lcrw_profile_count", "lcrw_table_chunk", "lcrw_table_bytes",
                "lcrw_table_operand_rows", "lcrw_refine_tau",
                "lcrw_reverse_panels_top_slots", "lcrw_plan_reverse_words_bound"}

# kernels each entry point launches (CUB-backed ones counted from an ncu launch list,
# profiles/); bench.py multiplies these by the per-step call counts for "gpu_launches".
KERNELS_PER_CALL = {
    "lcrw_max_sqnorm": 1, "lcrw_scale_from_max_sqnorm": 1, "lcrw_prepare_rows": 1, "lcrw_gather_rows": 1,
    "lcrw_row_classes": 13, "lcrw_match_rows": 2, "lcrw_restrict": 4, "lcrw_remap_ids": 1,
    "lcrw_segment_plan": 2, "lcrw_phase1": 1, "lcrw_zero_identical": 1, "lcrw_spmm": 1, "lcrw_spmm_dist": 1,
    "lcrw_topk_segments": 1, "lcrw_topk_sort": 7, "lcrw_topk_rows": 2,
    "lcrw_reverse_panels": 1, "lcrw_emd_batch": 1, "lcrw_symmetrize_max": 1, "lcrw_max_transposed": 1,
    "lcrw_max_transposed_into": 1, "lcrw_table_transpose": 1, "lcrw_table_min": 1,
    "lcrw_distance_table": 2, "lcrw_topk_sort_any": 7, "lcrw_squared_norms": 1, "lcrw_euclidean_f64": 1,
    "lcrw_segmented_min": 1, "lcrw_refine_near": 1, "lcrw_near_pairs_build": 7, "lcrw_near_scatter": 1,
    "lcrw_near_pairs_candidates": 1, "lcrw_near_pairs_finish": 6,
}
# lcrw_reverse_pipeline launches 7 kernels per doc batch (gather, 2 plan, phase1, zeros, refine,
# reverse_panels) in GEMM mode, 3 (table_min, refine, reverse_panels) with a distance table, plus the
# near-pair scatter when near pairs are given; bench.py adds those from the batch count (= its
# reverse_panels launches).
REVERSE_KERNELS_PER_BATCH = 7
REVERSE_KERNELS_PER_BATCH_TABLE = 3

CALLS: dict[str, int] = {}

_lib = None
_lock = threading.Lock()


class LcrwError(RuntimeError):
    """CUDA-side failure reported through the C ABI."""


def load() -> C.CDLL:
    """Load (once) and type the library; raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1711_07227_b200._build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def launches(calls: dict[str, int]) -> int:
    """Kernel launches implied by a call-count snapshot."""
    return sum(KERNELS_PER_CALL.get(n, 0) * c for n, c in calls.items())


def profile_reset(enable: bool) -> None:
    call("lcrw_profile_reset", 1 if enable else 0)


def profile_read() -> dict[str, dict[str, float]]:
    """name -> {ms, launches} of the native launch profiler (waits on the events)."""
    lib = load()
    out: dict[str, dict[str, float]] = {}
    buf = C.create_string_buffer(64)
    ms = C.c_float(0.0)
    for i in range(int(lib.lcrw_profile_count())):
        call("lcrw_profile_get", i, buf, 64, C.byref(ms))
        d = out.setdefault(buf.value.decode(), {"ms": 0.0, "launches": 0})
        d["ms"] += ms.value
        d["launches"] += 1
    return out


def value(name: str, *args):
    return getattr(load(), name)(*args)


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise on failure."""
    lib = load()
    CALLS[name] = CALLS.get(name, 0) + 1
    st = getattr(lib, name)(*args)
    if st == 0:
        return
    msg = (lib.lcrw_last_error() or b"").decode(errors="replace")
    if st == 1:
        raise ValueError(msg)
    if st == 3:
        raise NotImplementedError(f"{name}: {msg}")
    raise LcrwError(f"{name}: {msg}")
