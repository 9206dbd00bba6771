"""ctypes binding of libchebpr_b200.so (include/chebpr_cuda.h).

The library is the product: there is no CPU fallback.  Importing this module
fails loudly when the shared object has not been built; calls that need a GPU
fail with ``CudaError`` when none is visible.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libchebpr_b200.so")

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)


class cheb_build_opts(C.Structure):
    _fields_ = [("dedup", C.c_int), ("drop_isolated", C.c_int), ("n_hint", C.c_int64),
                ("device", C.c_int), ("row_ptr_64", C.c_int)]


class cheb_graph_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("nnz", C.c_int64),
                ("duplicates_removed", C.c_int64), ("isolated_dropped", C.c_int64),
                ("max_degree", C.c_int64), ("min_degree", C.c_int64), ("multi", C.c_int),
                ("row_ptr_64", C.c_int), ("inv_degree_array", C.c_int), ("device", C.c_int)]


class cheb_cpaa_opts(C.Structure):
    _fields_ = [("c", C.c_double), ("rounds", C.c_int), ("eps", C.c_double),
                ("max_rounds", C.c_int), ("parallelism", C.c_int), ("mode", C.c_int),
                ("precision", C.c_int), ("R", C.c_int), ("personalization", F64P),
                ("trace", C.c_int)]


class cheb_trace_row(C.Structure):
    _fields_ = [("k", C.c_int), ("c_k", C.c_double), ("S_k", C.c_double),
                ("residual_mass", C.c_double), ("l1_change", C.c_double),
                ("elapsed_ms", C.c_double), ("mass_T", C.c_double), ("err", C.c_double),
                ("err_l1", C.c_double)]


class cheb_load_opts(C.Structure):
    _fields_ = [("dedup", C.c_int), ("drop_isolated", C.c_int), ("symmetrize", C.c_int),
                ("device", C.c_int), ("row_ptr_64", C.c_int)]


class cheb_graph_stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("avg_degree", C.c_double),
                ("min_degree", C.c_int64), ("max_degree", C.c_int64), ("self_loops", C.c_int64),
                ("duplicates_removed", C.c_int64), ("isolated_dropped", C.c_int64),
                ("lines", C.c_int64), ("weights_ignored", C.c_int)]


class cheb_power_opts(C.Structure):
    _fields_ = [("c", C.c_double), ("rounds", C.c_int), ("tol", C.c_double),
                ("max_rounds", C.c_int), ("parallelism", C.c_int), ("mode", C.c_int)]


# name -> (restype, argtypes)
PEER_EXPORT_BYTES = 384  # CHEB_PEER_EXPORT_BYTES

_SIGS = {
    "cheb_last_error": (C.c_char_p, []),
    "cheb_version": (C.c_char_p, []),
    "cheb_device_count": (C.c_int, []),
    "cheb_beta": (C.c_int, [C.c_double, F64P]),
    "cheb_sigma": (C.c_int, [C.c_double, F64P]),
    "cheb_err_bound": (C.c_int, [C.c_double, C.c_int, F64P]),
    "cheb_plan_iterations": (C.c_int, [C.c_double, C.c_double, IP, F64P]),
    "cheb_coefficients": (C.c_int, [C.c_double, C.c_int, F64P, F64P, F64P]),
    "cheb_resolve_rounds": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_int, IP]),
    "cheb_kahan_sum": (C.c_double, [F64P, C.c_int64]),
    "cheb_build_opts_default": (None, [C.POINTER(cheb_build_opts)]),
    "cheb_graph_build": (C.c_int, [I64P, C.c_int64, C.POINTER(cheb_build_opts),
                                   C.POINTER(C.c_void_p), C.POINTER(cheb_graph_info)]),
    "cheb_graph_build_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_int,
                                          C.POINTER(cheb_build_opts), C.POINTER(C.c_void_p),
                                          C.POINTER(cheb_graph_info)]),
    "cheb_graph_upload_csr": (C.c_int, [I64P, C.c_int64, I64P, C.c_int64, I64P, C.c_int64,
                                        F64P, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                        C.c_int, C.POINTER(C.c_void_p)]),
    "cheb_graph_download_csr": (C.c_int, [C.c_void_p, I64P, I64P, I64P]),
    "cheb_load_opts_default": (None, [C.POINTER(cheb_load_opts)]),
    "cheb_graph_load_edge_list": (C.c_int, [C.c_char_p, C.POINTER(cheb_load_opts), C.POINTER(C.c_void_p),
                                            C.POINTER(cheb_graph_stats)]),
    "cheb_graph_load_matrix_market": (C.c_int, [C.c_char_p, C.POINTER(cheb_load_opts), C.POINTER(C.c_void_p),
                                                C.POINTER(cheb_graph_stats)]),
    "cheb_graph_parse_text": (C.c_int, [C.c_char_p, C.c_int64, C.c_int, C.c_char_p, C.POINTER(cheb_load_opts),
                                        C.POINTER(C.c_void_p), C.POINTER(cheb_graph_stats)]),
    "cheb_graph_validate_stats": (C.c_int, [C.c_void_p, C.POINTER(cheb_graph_stats)]),
    "cheb_validate_csr": (C.c_int, [I64P, C.c_int64, I64P, C.c_int64, I64P, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int, C.c_int64, C.c_int64, C.c_int, C.POINTER(cheb_graph_stats)]),
    "cheb_graph_get_info": (C.c_int, [C.c_void_p, C.POINTER(cheb_graph_info)]),
    "cheb_graph_free": (None, [C.c_void_p]),
    "cheb_partition_vertices": (C.c_int, [I64P, C.c_int64, C.c_int, I64P]),
    "cheb_partition_plan": (C.c_int, [I64P, C.c_int64, C.c_int, I64P, I64P, I64P]),
    "cheb_cpaa_opts_default": (None, [C.POINTER(cheb_cpaa_opts)]),
    "cheb_cpaa": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), F64P, C.c_int64, F64P,
                            C.POINTER(cheb_trace_row), IP, F64P]),
    "cheb_cpaa_device": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts),
                                   C.POINTER(C.c_void_p), C.c_int]),
    "cheb_last_timing": (C.c_int, [C.c_void_p, F64P, F64P, IP, IP]),
    "cheb_set_tuning": (C.c_int, [C.c_char_p, C.c_int]),
    "cheb_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int]),
    "cheb_comm_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "cheb_comm_destroy": (None, [C.c_void_p]),
    "cheb_graph_attach_comm": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cheb_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p)]),
    "cheb_group_cpaa": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), F64P, C.POINTER(cheb_trace_row), IP,
                                  F64P]),
    "cheb_group_profile": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), F64P, C.c_int]),
    "cheb_group_destroy": (None, [C.c_void_p]),
    "cheb_graph_view_bins": (C.c_int, [C.c_void_p, I64P, I64P, I64P]),
    "cheb_peer_export": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]),
    "cheb_peer_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "cheb_peer_detach": (C.c_int, [C.c_void_p]),
    "cheb_graph_partition_info": (C.c_int, [C.c_void_p, I64P, I64P, I64P, I64P]),
    "cheb_graph_exchange_info": (C.c_int, [C.c_void_p, I64P, I64P]),
    "cheb_partition_block_rows": (C.c_int, []),
    "cheb_graph_view_download": (C.c_int, [C.c_void_p, I64P, I64P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), I64P]),
    "cheb_graph_view_windows": (C.c_int, [C.c_void_p, I64P, C.POINTER(C.c_uint16), C.POINTER(C.c_uint16),
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "cheb_graph_view_tiles": (C.c_int, [C.c_void_p, I64P, I64P, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32)]),
    "cheb_cpaa_batch": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), I64P, F64P, F64P,
                                  C.POINTER(cheb_trace_row), IP]),
    "cheb_cpaa_batch_profile": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), I64P, F64P, C.c_int,
                                          IP]),
    "cheb_cpaa_profile": (C.c_int, [C.c_void_p, C.POINTER(cheb_cpaa_opts), F64P, C.c_int, IP]),
    "cheb_power_opts_default": (None, [C.POINTER(cheb_power_opts)]),
    "cheb_power": (C.c_int, [C.c_void_p, C.POINTER(cheb_power_opts), F64P, C.c_int64, F64P,
                             C.POINTER(cheb_trace_row), C.c_int, IP, F64P]),
    "cheb_transition_apply": (C.c_int, [C.c_void_p, F64P, C.c_int64, F64P, C.c_int]),
    "cheb_state_init": (C.c_int, [C.c_void_p, C.c_double, C.c_int]),
    "cheb_state_set": (C.c_int, [C.c_void_p, F64P, F64P, F64P, C.c_int]),
    "cheb_state_generate": (C.c_int, [C.c_void_p]),
    "cheb_state_accumulate": (C.c_int, [C.c_void_p, C.c_double]),
    "cheb_state_rotate": (C.c_int, [C.c_void_p]),
    "cheb_state_get": (C.c_int, [C.c_void_p, F64P, F64P, F64P, F64P, IP]),
    "cheb_gen_ring": (C.c_int, [C.c_int64, C.POINTER(I64P), I64P]),
    "cheb_gen_star": (C.c_int, [C.c_int64, C.POINTER(I64P), I64P]),
    "cheb_gen_regular": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(I64P), I64P]),
    "cheb_gen_gnp": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, C.POINTER(I64P), I64P]),
    "cheb_gen_rmat": (C.c_int, [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                C.c_int, C.c_int, C.POINTER(C.c_void_p), I64P]),
    "cheb_gen_chung_lu": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64,
                                    C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_void_p), I64P]),
    "cheb_gen_last_error": (C.c_char_p, []),
    "cheb_free": (None, [C.c_void_p]),
    "cheb_device_free": (None, [C.c_void_p, C.c_int]),
}

# Symbols declared in include/*.h (checked by tests/test_capi_symbols.py).
EXPORTED = sorted(_SIGS)

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the C-ABI library.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make` (the CUDA library is required; there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
