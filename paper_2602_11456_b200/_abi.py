"""ctypes declarations of include/sparsedelta.h (argument marshalling only).

Loads the in-tree ``libsparsedelta.so`` built by ``__graft_entry__.build()``.  There is
no fallback: if the library is missing or fails to load, importing the binding's
compute entry points raises.
"""

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARSEDELTA_LIB") or os.path.join(HERE, "libsparsedelta.so")  # override: A/B runs only

DELTA_OK, DELTA_EINVAL, DELTA_ESHAPE, DELTA_ECAPACITY = 0, -1, -2, -3
DELTA_ECORRUPT, DELTA_ENAME, DELTA_ECUDA, DELTA_ENOMEM = -4, -5, -6, -7
DELTA_ELEM16, DELTA_ELEM32 = 0, 1

STATUS_NAMES = {0: "OK", -1: "EINVAL", -2: "ESHAPE", -3: "ECAPACITY", -4: "ECORRUPT",
                -5: "ENAME", -6: "ECUDA", -7: "ENOMEM",
                -8: "EAGAIN"}
DELTA_EAGAIN = -8
DETAIL_NAMES = {0: None, 1: "truncated", 2: "overlong", 3: "overflow", 4: "nonincreasing",
                5: "range", 6: "count", 7: "name", 8: "numel", 9: "mode", 10: "layout"}

# Every symbol include/sparsedelta.h declares (tests/test_abi.py checks the export list).
EXPORTS = ("delta_ctx_create", "delta_ctx_destroy", "delta_last_error", "delta_last_detail",
           "delta_version", "delta_size", "delta_extract", "delta_apply", "delta_set_profiling",
           "delta_last_timing", "delta_apply_async", "delta_apply_wait", "delta_set_option",
           "delta_apply_async_dev", "delta_table_dev", "delta_assemble", "delta_assemble_wait",
           "delta_digest", "delta_extract_async", "delta_extract_wait", "delta_apply_async_chain",
           "delta_merge", "delta_timing_totals", "delta_record_sizes", "delta_assemble_records",
           "delta_size_table", "delta_compute_rho", "delta_table_rebase",
           "delta_extract_scan_async", "delta_extract_emit_async",
           "delta_container_header")
DELTA_OPT_APPLY_CTAS_PER_SM, DELTA_OPT_EMIT_CTAS_PER_SM, DELTA_OPT_SCAN_KERNEL = 1, 2, 3
DELTA_OPT_SCATTER_CTAS_PER_SM, DELTA_OPT_PREFETCH_TILES, DELTA_OPT_SCATTER_ORDER, DELTA_OPT_MODE = 4, 5, 6, 7
DELTA_OPT_INDEX_CODEC = 8  # 1 LEB128 gaps (default), 2 fixed-width absolute indices (reading R18)
DELTA_OPT_ADVANCE = 9      # 2: extract-and-advance (old spans overwritten with new; NEXT f3)
DELTA_OPT_ASSEMBLE_CTAS = 10  # CTAs of the NVLink assembly kernels


class Span(ctypes.Structure):
    _fields_ = [("old_dev", c_void_p), ("new_dev", c_void_p), ("numel", c_uint64)]


class Tensor(ctypes.Structure):
    _fields_ = [("name", c_char_p), ("name_len", c_uint32), ("n_spans", c_uint32),
                ("spans", POINTER(Span))]


class Target(ctypes.Structure):
    _fields_ = [("w_dev", c_void_p), ("numel", c_uint64), ("name", c_char_p), ("name_len", c_uint32)]


class RecordInfo(ctypes.Structure):
    _fields_ = [("record_offset", c_uint64), ("element_count", c_uint64), ("nnz", c_uint64),
                ("index_offset", c_uint64), ("index_bytes", c_uint64), ("values_offset", c_uint64),
                ("record_bytes", c_uint64)]


class Timing(ctypes.Structure):
    _fields_ = [(f, ctypes.c_float) for f in (
        "scan_ms", "lens_ms", "finalize_ms", "emit_ms", "headers_ms", "locate_ms", "decode_ms",
        "apply_scan_ms", "scatter_ms")]


_lib = None


def lib():
    """The loaded library (loaded once).  Raises if it is missing: no CPU fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build() (there is no "
                               "fallback implementation)")
        L = ctypes.CDLL(LIB_PATH)
        L.delta_ctx_create.argtypes = [POINTER(c_void_p), c_int]
        L.delta_ctx_create.restype = c_int
        L.delta_ctx_destroy.argtypes = [c_void_p]
        L.delta_ctx_destroy.restype = None
        L.delta_last_error.argtypes = [c_void_p]
        L.delta_last_error.restype = c_char_p
        L.delta_last_detail.argtypes = [c_void_p]
        L.delta_last_detail.restype = c_int
        L.delta_version.argtypes = []
        L.delta_version.restype = c_char_p
        L.delta_size.argtypes = [c_void_p, POINTER(Tensor), c_uint32, c_int, c_void_p, POINTER(c_uint64)]
        L.delta_size.restype = c_int
        L.delta_size_table.argtypes = [c_void_p, c_uint32, POINTER(RecordInfo), c_void_p]
        L.delta_size_table.restype = c_int
        L.delta_compute_rho.argtypes = [c_void_p, POINTER(Tensor), c_uint32, c_int, c_void_p, POINTER(c_uint64),
                                        POINTER(c_uint64), POINTER(c_uint64), POINTER(ctypes.c_double)]
        L.delta_compute_rho.restype = c_int
        L.delta_table_rebase.argtypes = [POINTER(RecordInfo), c_uint32, c_uint64]
        L.delta_table_rebase.restype = c_int
        L.delta_extract_scan_async.argtypes = [c_void_p, POINTER(Tensor), c_uint32, c_int, c_void_p, c_void_p]
        L.delta_extract_scan_async.restype = c_int
        L.delta_extract_emit_async.argtypes = [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_uint64, c_void_p,
                                               c_uint32, c_uint32, c_void_p]
        L.delta_extract_emit_async.restype = c_int
        L.delta_container_header.argtypes = [c_void_p, c_void_p, c_uint64, c_uint64, c_uint64, c_int, c_uint32, c_int,
                                             c_void_p, c_void_p]
        L.delta_container_header.restype = c_int
        L.delta_extract.argtypes = [c_void_p, POINTER(Tensor), c_uint32, c_int, c_void_p, c_uint64,
                                    POINTER(RecordInfo), c_void_p, POINTER(c_uint64)]
        L.delta_extract.restype = c_int
        L.delta_apply.argtypes = [c_void_p, POINTER(Target), c_uint32, c_int, c_void_p, c_uint64,
                                  POINTER(RecordInfo), c_void_p]
        L.delta_apply.restype = c_int
        L.delta_apply_async.argtypes = L.delta_apply.argtypes
        L.delta_apply_async.restype = c_int
        L.delta_apply_async_dev.argtypes = [c_void_p, POINTER(Target), c_uint32, c_int, c_void_p, c_uint64,
                                            c_void_p, c_void_p]
        L.delta_apply_async_dev.restype = c_int
        L.delta_extract_async.argtypes = [c_void_p, POINTER(Tensor), c_uint32, c_int, c_void_p, c_uint64,
                                          c_void_p, c_void_p]
        L.delta_extract_async.restype = c_int
        L.delta_extract_wait.argtypes = [c_void_p, POINTER(c_uint64)]
        L.delta_extract_wait.restype = c_int
        L.delta_apply_async_chain.argtypes = [c_void_p, POINTER(Target), c_uint32, c_int, c_void_p, c_uint64,
                                              c_void_p, c_void_p, c_void_p]
        L.delta_apply_async_chain.restype = c_int
        L.delta_table_dev.argtypes = [c_void_p]
        L.delta_table_dev.restype = c_void_p
        L.delta_assemble.argtypes = [c_void_p, c_void_p, c_void_p, c_uint64, c_void_p, c_uint32, c_uint32,
                                     c_void_p]
        L.delta_assemble.restype = c_int
        L.delta_assemble_wait.argtypes = [c_void_p, c_void_p]
        L.delta_assemble_wait.restype = c_int
        L.delta_digest.argtypes = [c_void_p, c_void_p, c_uint64, ctypes.c_char_p, c_void_p]
        L.delta_digest.restype = c_int
        L.delta_merge.argtypes = [c_void_p, ctypes.c_uint32, c_int, c_void_p, c_uint64, c_void_p, c_uint64,
                                  c_void_p, c_uint64, c_void_p, ctypes.POINTER(c_uint64)]
        L.delta_merge.restype = c_int
        L.delta_timing_totals.argtypes = [c_void_p, c_void_p, ctypes.POINTER(ctypes.c_uint32)]
        L.delta_timing_totals.restype = c_int
        L.delta_record_sizes.argtypes = [c_void_p, c_void_p, ctypes.c_uint32, c_void_p, c_void_p, ctypes.c_uint32,
                                         c_void_p]
        L.delta_record_sizes.restype = c_int
        L.delta_assemble_records.argtypes = [c_void_p, c_void_p, c_void_p, ctypes.c_uint32, c_void_p, ctypes.c_uint32,
                                             c_void_p, c_uint64, c_void_p]
        L.delta_assemble_records.restype = c_int
        L.delta_apply_wait.argtypes = [c_void_p, c_void_p]
        L.delta_apply_wait.restype = c_int
        L.delta_set_option.argtypes = [c_void_p, c_int, ctypes.c_int64]
        L.delta_set_option.restype = c_int
        L.delta_set_profiling.argtypes = [c_void_p, c_int]
        L.delta_set_profiling.restype = c_int
        L.delta_last_timing.argtypes = [c_void_p, POINTER(Timing)]
        L.delta_last_timing.restype = c_int
        _lib = L
    return _lib
