"""ctypes binding of libsel.so (include/sel.h) — argument marshalling only. Every step of the
probe runs inside the library; there is no Python or CPU fallback: if the library is missing
the import fails loudly."""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEL_LIB") or os.path.join(HERE, "libsel.so")

SEL_OK, SEL_E_ARG, SEL_E_ALIGN, SEL_E_TYPE, SEL_E_PROGRAM, SEL_E_TOO_LARGE, SEL_E_CUDA, \
    SEL_E_NCCL, SEL_E_STATE = range(9)
SEL_ERR = (1 << 64) - 1
SEL_KEEP_SELECTION = 1
SEL_PD_CODED, SEL_PD_WHOLE_CHUNKS, SEL_PD_CONSTANT, SEL_PD_KEPT_VALUES = 1, 2, 4, 8
STATUS_NAMES = {0: "SEL_OK", 1: "SEL_E_ARG", 2: "SEL_E_ALIGN", 3: "SEL_E_TYPE",
                4: "SEL_E_PROGRAM", 5: "SEL_E_TOO_LARGE", 6: "SEL_E_CUDA", 7: "SEL_E_NCCL",
                8: "SEL_E_STATE"}

# Every symbol include/sel.h declares (tests check the library exports exactly these).
EXPORTS = ["sel_ctx_create", "sel_ctx_set_comm", "sel_nccl_unique_id", "sel_ctx_destroy",
           "sel_ctx_peer_handle", "sel_ctx_set_peers", "sel_ctx_set_peer_timeout",
           "sel_ctx_export_buffer",
           "sel_ctx_import_buffer", "sel_execute_to",
           "sel_ctx_set_timing", "sel_ctx_set_option", "sel_ctx_last_kernel_ms", "sel_table_register",
           "sel_table_release", "sel_count", "sel_count_async", "sel_count_ex", "sel_execute", "sel_pushdown",
           "sel_ctx_last_times", "sel_count_batch", "sel_count_sampled", "sel_histogram",
           "sel_bitmap_register", "sel_bitmap_release",
           "sel_prepare_execute", "sel_prepared_execute", "sel_prepared_execute_async",
           "sel_prepared_release",
           "sel_ctx_last_pushdown_path", "sel_ctx_last_pushdown_flags", "sel_ctx_set_pushdown_path", "sel_program_check",
           "sel_program_path", "sel_program_plan_json", "sel_last_error",
           "sel_last_error_message", "sel_abi_version", "sel_sample_estimate",
           "sel_equi_depth_estimate"]


class sel_column(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("data", ctypes.c_void_p), ("dict_size", ctypes.c_uint32)]


class SelError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsel.so not built at {LIB_PATH}: run `python -c 'import "
                          "__graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, u32, sz, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_int
    sig = {
        "sel_ctx_create": (i32, [i32, ctypes.POINTER(vp)]),
        "sel_ctx_set_comm": (i32, [vp, i32, i32, vp]),
        "sel_ctx_peer_handle": (i32, [vp, vp]),
        "sel_ctx_set_peers": (i32, [vp, i32, i32, vp]),
        "sel_ctx_set_peer_timeout": (i32, [vp, u64]),
        "sel_ctx_export_buffer": (i32, [vp, vp, vp]),
        "sel_ctx_import_buffer": (i32, [vp, vp, ctypes.POINTER(ctypes.c_void_p)]),
        "sel_nccl_unique_id": (i32, [vp]),
        "sel_ctx_destroy": (None, [vp]),
        "sel_ctx_set_timing": (i32, [vp, i32]),
        "sel_ctx_set_option": (i32, [vp, ctypes.c_char_p, ctypes.c_int64]),
        "sel_ctx_last_kernel_ms": (i32, [vp, ctypes.POINTER(ctypes.c_float)]),
        "sel_table_register": (i32, [vp, ctypes.POINTER(sel_column), u32, u64, u64, u64,
                                     ctypes.POINTER(vp)]),
        "sel_table_release": (None, [vp]),
        "sel_count": (u64, [vp, ctypes.c_char_p, sz, vp]),
        "sel_count_ex": (u64, [vp, ctypes.c_char_p, sz, u32, vp, u32, vp]),
        "sel_count_async": (i32, [vp, ctypes.c_char_p, sz, vp, vp]),
        "sel_histogram": (i32, [vp, u32, u32, u32, u32, vp, vp, vp, vp, vp, vp]),
        "sel_execute": (u64, [vp, ctypes.c_char_p, sz, vp, u32, u64, vp, vp, u64,
                              ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(i32), vp]),
        "sel_execute_to": (u64, [vp, ctypes.c_char_p, sz, vp, u32, u64, vp, vp, u64,
                                 ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(i32), vp]),
        "sel_count_sampled": (u64, [vp, ctypes.c_char_p, sz, u32, u32, ctypes.POINTER(u64), vp]),
        "sel_count_batch": (i32, [vp, vp, vp, u32, ctypes.POINTER(u64), vp]),
        "sel_bitmap_register": (i32, [vp, vp, u64, ctypes.POINTER(u32)]),
        "sel_bitmap_release": (i32, [vp, u32]),
        "sel_prepare_execute": (i32, [vp, ctypes.c_char_p, sz, vp, u32, u64, vp, vp, u64,
                                      ctypes.POINTER(vp)]),
        "sel_prepared_execute": (u64, [vp, ctypes.POINTER(u64), ctypes.POINTER(u64),
                                       ctypes.POINTER(i32), vp]),
        "sel_prepared_execute_async": (u64, [vp, ctypes.POINTER(u64), ctypes.POINTER(u64),
                                             ctypes.POINTER(i32), vp]),
        "sel_prepared_release": (None, [vp]),
        "sel_ctx_last_times": (i32, [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
        "sel_ctx_last_pushdown_path": (i32, [vp]),
        "sel_ctx_last_pushdown_flags": (i32, [vp]),
        "sel_ctx_set_pushdown_path": (i32, [vp, i32]),
        "sel_pushdown": (u64, [vp, ctypes.c_char_p, sz, vp, u32, vp, vp, u64,
                               ctypes.POINTER(u64), ctypes.POINTER(u64), vp]),
        "sel_program_check": (i32, [ctypes.c_char_p, sz, vp, u32]),
        "sel_program_path": (i32, [ctypes.c_char_p, sz, vp, u32]),
        "sel_program_plan_json": (ctypes.c_long, [ctypes.c_char_p, sz, vp, u32, vp, sz]),
        "sel_last_error": (i32, []),
        "sel_last_error_message": (ctypes.c_char_p, []),
        "sel_abi_version": (i32, []),
        "sel_sample_estimate": (ctypes.c_double, [u64, u64, u64]),
        "sel_equi_depth_estimate": (ctypes.c_double, [vp, vp, vp, u32, u64, ctypes.c_int64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def last_error() -> SelError:
    L = lib()
    return SelError(L.sel_last_error(), (L.sel_last_error_message() or b"").decode())


def check(status: int) -> None:
    if status != SEL_OK:
        raise last_error()
