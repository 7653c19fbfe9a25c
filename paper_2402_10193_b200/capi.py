"""ctypes binding of include/bitdelta/capi.h (libbitdelta_b200.so).

The product path: every function here forwards to the sm_100a kernels through
the C-ABI. There is no CPU fallback — a missing library or a non-B200 device
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BD_LIB") or os.path.join(HERE, "libbitdelta_b200.so")  # BD_LIB: A/B experiments

u64 = C.c_uint64
vp = C.c_void_p

# 1 + deltakit::errc (P:include/deltakit/error.hpp:10-25)
ERRC = {
    1: "io", 2: "malformed_header", 3: "json_parse", 4: "bad_offsets", 5: "unsupported_dtype",
    6: "shape_mismatch", 7: "name_mismatch", 8: "length_mismatch", 9: "bad_argument",
    10: "bad_token", 11: "non_finite", 12: "no_convergence", 13: "duplicate_id", 14: "unknown_id",
    100: "cuda", 101: "no_device", 102: "unsupported_device",
}
BD_F32, BD_BF16 = 0, 1


class BitDeltaError(RuntimeError):
    """Mirror of deltakit::Error (error.hpp:27-42): carries the errc category."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.code = ERRC.get(status, str(status))
        super().__init__(f"[{self.code}] {msg}")


class CompressJob(C.Structure):
    _fields_ = [("base", vp), ("fine", vp), ("rows", u64), ("cols", u64), ("bits", vp), ("alpha", vp)]


class Arch(C.Structure):
    _fields_ = [("vocab", u64), ("dim", u64), ("kv_dim", u64), ("n_layers", u64), ("n_heads", u64),
                ("intermediate", u64), ("max_seq", u64), ("rope_theta", C.c_float)]


class DeltaEntry(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int), ("rows", u64), ("cols", u64), ("planes", u64),
                ("bits", vp), ("scales", C.POINTER(C.c_float)), ("raw", vp), ("is_device", C.c_int)]


class Request(C.Structure):
    _fields_ = [("request_id", u64), ("token", C.c_int32), ("position", u64)]


class PoolStats(C.Structure):
    _fields_ = [("backbone_passes", u64), ("cold_loads", u64), ("last_cold_load_ms", C.c_double),
                ("resident_bytes", u64), ("kernels_last_step", u64), ("delta_paths", C.c_char * 8)]


SYMBOLS = [
    "bd_abi_version", "bd_last_error", "bd_device_check", "bd_launch_count", "bd_packed_size",
    "bd_compress", "bd_compress_batched", "bd_compress_stack", "bd_packed_signed_accumulate",
    "bd_packed_matvec", "bd_packed_signed_accumulate_t", "bd_delta_linear_backward", "bd_rtn_quantize", "bd_int8_matmul_nt", "bd_pool_set_tensor_i8", "bd_multitenant_linear", "bd_multitenant_linear_f32", "bd_pool_create", "bd_pool_destroy",
    "bd_pool_set_tensor", "bd_pool_register_delta", "bd_pool_register_delta_file",
    "bd_bdelta_validate", "bd_pool_open_request", "bd_pool_close_request", "bd_pool_decode_step",
    "bd_pool_decode_layers", "bd_pool_get_stats", "bd_pool_profile_layers", "bd_pool_profile_layers_serial", "bd_nccl_unique_id",
    "bd_pool_init_comm", "bd_pool_init_loopback", "bd_trace_enable", "bd_trace_read",
]


@lru_cache(maxsize=None)
def lib() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} is missing — build it with `python -m paper_2402_10193_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.bd_last_error.restype = C.c_char_p
    L.bd_launch_count.restype = u64
    L.bd_packed_size.restype = u64
    L.bd_packed_size.argtypes = [u64, u64]
    L.bd_compress.argtypes = [vp, vp, C.c_int, u64, u64, vp, vp, vp]
    L.bd_compress_batched.argtypes = [C.POINTER(CompressJob), C.c_int, C.c_int, vp]
    L.bd_compress_stack.argtypes = [vp, vp, C.c_int, u64, u64, u64, vp, vp, vp]
    L.bd_packed_signed_accumulate.argtypes = [vp, u64, u64, vp, u64, vp, vp]
    L.bd_packed_matvec.argtypes = [vp, C.c_float, u64, u64, vp, u64, vp, vp]
    L.bd_packed_signed_accumulate_t.argtypes = [vp, u64, u64, vp, u64, vp, vp]
    L.bd_rtn_quantize.argtypes = [vp, u64, u64, vp, vp, vp]
    L.bd_int8_matmul_nt.argtypes = [vp, u64, u64, vp, vp, u64, vp, vp]
    L.bd_delta_linear_backward.argtypes = [C.c_int32, C.POINTER(vp), C.POINTER(C.c_float), u64, u64, vp, u64,
                                           C.POINTER(vp), vp, vp, vp]
    L.bd_multitenant_linear.argtypes = [vp, u64, u64, C.c_int32, C.POINTER(vp), C.POINTER(C.c_float),
                                        C.c_int32, C.POINTER(C.c_int32), vp, vp, vp]
    L.bd_multitenant_linear_f32.argtypes = L.bd_multitenant_linear.argtypes
    L.bd_pool_create.argtypes = [C.POINTER(Arch), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.bd_pool_destroy.argtypes = [vp]
    L.bd_pool_destroy.restype = None
    L.bd_pool_set_tensor.argtypes = [vp, C.c_char_p, vp, C.c_int, C.c_int, u64, u64]
    L.bd_pool_set_tensor_i8.argtypes = [vp, C.c_char_p, vp, vp, C.c_int, u64, u64]
    L.bd_pool_register_delta.argtypes = [vp, C.c_char_p, C.POINTER(DeltaEntry), C.c_int]
    L.bd_pool_register_delta_file.argtypes = [vp, C.c_char_p, C.c_char_p, C.c_int]
    L.bd_pool_open_request.argtypes = [vp, C.c_char_p, C.POINTER(u64)]
    L.bd_pool_close_request.argtypes = [vp, u64]
    L.bd_pool_decode_step.argtypes = [vp, C.POINTER(Request), u64, C.c_int, vp, vp]
    L.bd_pool_decode_layers.argtypes = [vp, C.POINTER(Request), u64, vp, vp, vp]
    L.bd_pool_get_stats.argtypes = [vp, C.POINTER(PoolStats)]
    L.bd_pool_profile_layers.argtypes = [vp, C.POINTER(Request), u64, vp, vp, C.POINTER(C.c_double),
                                         C.POINTER(u64), vp]
    L.bd_pool_profile_layers_serial.argtypes = L.bd_pool_profile_layers.argtypes
    L.bd_bdelta_validate.argtypes = [C.c_char_p, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]
    L.bd_nccl_unique_id.argtypes = [vp]
    L.bd_pool_init_comm.argtypes = [vp, vp]
    L.bd_pool_init_loopback.argtypes = [vp, C.c_char_p]
    if hasattr(L, "bd_trace_enable"):  # diagnostics (absent from older builds used in A/B runs)
        L.bd_trace_enable.argtypes = [C.c_uint32]
        L.bd_trace_read.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint32)]
    return L


def check(status: int) -> None:
    if status != 0:
        raise BitDeltaError(status, lib().bd_last_error().decode(errors="replace"))
