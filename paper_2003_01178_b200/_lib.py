"""ctypes binding of the C ABI in include/crystal_b200.h.

The product path has exactly one implementation: libcrystal_b200.so (sm_100a
CUDA kernels).  If the library is missing this module raises at import time;
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcrystal_b200.so")

CRYS_OK, CRYS_ECONFIG, CRYS_ECONTRACT, CRYS_EBUILD, CRYS_EIO, CRYS_ECUDA, CRYS_ENOTBUILT, CRYS_ENCCL = range(8)
CRYS_PARTIAL_HEADER = 32
CRYS_LT, CRYS_LE, CRYS_GT, CRYS_GE, CRYS_EQ, CRYS_BETWEEN = range(6)
CRYS_ORDER_INPUT, CRYS_ORDER_CRYSTAL = 0, 1
CRYS_SORT_LSB, CRYS_SORT_MSB = 0, 1
CRYS_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class crys_pred(C.Structure):
    _fields_ = [("op", C.c_int32), ("lo", C.c_int32), ("hi", C.c_int32)]


class crys_group_box(C.Structure):
    _fields_ = [("nparts", C.c_int32), ("lo", C.c_int32 * 3), ("card", C.c_int32 * 3), ("pad", C.c_int32),
                ("cells", C.c_int64)]


class crys_host_column(C.Structure):
    _fields_ = [("table", C.c_char_p), ("column", C.c_char_p), ("h_data", C.c_void_p),
                ("rows", C.c_int64)]


# (name, restype, argtypes) for every exported symbol of crystal_b200.h
_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
SIGNATURES = [
    ("crys_last_error", C.c_char_p, []),
    ("crys_version", C.c_char_p, []),
    ("crys_init", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("crys_init_group", C.c_int, [C.c_int, _I32P, C.POINTER(_P)]),
    ("crys_group_shards", C.c_int, [_P]),
    ("crys_group_devices", C.c_int, [_P]),
    ("crys_group_uses_nccl", C.c_int, [_P]),
    ("crys_nccl_version", C.c_char_p, []),
    ("crys_device_count", C.c_int, []),
    ("crys_destroy", None, [_P]),
    ("crys_set_stream", C.c_int, [_P, _P]),
    ("crys_synchronize", C.c_int, [_P]),
    ("crys_kernel_launches", C.c_int64, [_P]),
    ("crys_db_generate", C.c_int, [_P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.POINTER(_P)]),
    ("crys_device_alloc", C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    ("crys_device_free", None, [_P, _P]),
    ("crys_copy_to_device", C.c_int, [_P, _P, _P, C.c_size_t]),
    ("crys_copy_to_host", C.c_int, [_P, _P, _P, C.c_size_t]),
    ("crys_fill_uniform_i32", C.c_int, [_P, _P, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
                                        C.c_int32, C.c_int32]),
    ("crys_fill_float_pairs", C.c_int, [_P, _P, _P, C.c_int64, C.c_uint64, C.c_uint64, C.c_float,
                                        C.c_float]),
    ("crys_db_create", C.c_int, [_P, C.c_int64, C.c_uint64, C.POINTER(_P)]),
    ("crys_db_upload_column", C.c_int, [_P, C.c_char_p, C.c_char_p, _P, C.c_int64]),
    ("crys_db_upload_host", C.c_int, [_P, C.POINTER(crys_host_column), C.c_int]),
    ("crys_db_load_column_file", C.c_int, [_P, C.c_char_p, C.c_char_p, C.c_char_p]),
    ("crys_db_save_column_file", C.c_int, [_P, C.c_char_p, C.c_char_p, C.c_char_p]),
    ("crys_db_column", C.c_int, [_P, C.c_char_p, C.c_char_p, C.POINTER(_P), _I64P]),
    ("crys_db_download_column", C.c_int, [_P, C.c_char_p, C.c_char_p, _P, C.c_int64]),
    ("crys_db_column_rows", C.c_int, [_P, C.c_char_p, C.c_char_p, _I64P]),
    ("crys_db_free", None, [_P]),
    ("crys_query_shape", C.c_int, [C.c_int, _I64P, _I32P, _I32P]),
    ("crys_query_plan_json", C.c_int, [C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("crys_run_query", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int64, _I64P, _P]),
    ("crys_run_query_host", C.c_int, [_P, C.POINTER(crys_host_column), C.c_int, C.c_int, C.c_int,
                                      C.c_int, _P, _P, C.c_int64, _I64P, _P]),
    ("crys_query_partial", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("crys_query_partial_box", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, C.c_int64, _I64P,
                                         C.POINTER(crys_group_box)]),
    ("crys_query_finalize_box", C.c_int, [_P, C.c_int, C.POINTER(crys_group_box), _P, _P, _P, C.c_int64,
                                          _I64P, _P]),
    ("crys_query_finalize", C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int64, _I64P, _P]),
    ("crys_query_finalize_host", C.c_int, [C.c_int, _P, _P, _P, _P, C.c_int64, _I64P, _P]),
    ("crys_select_i32", C.c_int, [_P, _P, C.c_int64, crys_pred, _P, _I64P, C.c_int, C.c_int, C.c_int]),
    ("crys_block_ops_run", C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_int, crys_pred, _P, _P, _P, _P, _P]),
    ("crys_project_f32", C.c_int, [_P, _P, _P, C.c_int64, C.c_float, C.c_float, _P, C.c_int,
                                   C.c_int, C.c_int]),
    ("crys_ht_build", C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, C.POINTER(_P)]),
    ("crys_ht_upload", C.c_int, [_P, _P, _P, C.c_int64, C.POINTER(_P)]),
    ("crys_ht_download", C.c_int, [_P, _P, _P]),
    ("crys_ht_capacity", C.c_int64, [_P]),
    ("crys_ht_free", None, [_P]),
    ("crys_join_probe_sum", C.c_int, [_P, _P, _P, C.c_int64, _P, C.c_int, C.c_int, _I64P]),
    ("crys_sort_pairs", C.c_int, [_P, _P, _P, C.c_int64, C.c_int, C.c_int]),
    ("crys_radix_histogram", C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_int, C.c_int64, _P]),
    ("crys_radix_partition", C.c_int, [_P, _P, _P, C.c_int64, C.c_int, C.c_int, _P, _P]),
    ("crys_stream_read_gbs", C.c_int, [_P, _P, C.c_size_t, C.c_int, C.POINTER(C.c_double)]),
    ("crys_last_timing", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("crys_enable_timing", C.c_int, [_P, C.c_int]),
]


def _torch_nccl():
    """The libnccl.so.2 of the nvidia-nccl wheel torch links against (found
    without importing torch).  The library dlopens NCCL lazily; pointing it
    here keeps ONE NCCL per process whichever of torch / this library loads
    it first (a second, older libnccl.so.2 would break torch's import)."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


def _load() -> C.CDLL:
    if "CRYS_NCCL_LIBRARY" not in os.environ:
        p = _torch_nccl()
        if p:
            os.environ["CRYS_NCCL_LIBRARY"] = p
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 kernels are not built "
            "(run `make lib` or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
