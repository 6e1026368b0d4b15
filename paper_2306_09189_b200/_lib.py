"""ctypes binding of libfheconv.so (the C ABI in include/fheconv.h).

No fallback: if the shared library is missing or fails to load, importing
this module raises. fhe_ctx_create itself fails with FHE_E_CUDA when no
sm_100 GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FHECONV_LIB") or os.path.join(PKG, "libfheconv.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)
vp = C.c_void_p
vpp = C.POINTER(C.c_void_p)

FHE_OK, FHE_E_INVALID, FHE_E_RUNTIME, FHE_E_CUDA, FHE_E_NOKEY = 0, -1, -2, -3, -4


class FheParams(C.Structure):
    _fields_ = [("log_n", C.c_int), ("n_q", C.c_int), ("q_bits", C.POINTER(C.c_int)), ("n_p", C.c_int),
                ("p_bits", C.POINTER(C.c_int)), ("log_scale", C.c_int), ("device", C.c_int)]


LEDGER_FIELDS = ["rotations", "hoisted_rotations", "hoist_groups", "ct_pt_mults", "ct_ct_mults", "adds",
                 "bootstraps", "max_depth_consumed", "distinct_amounts", "key_switches", "modups", "moddowns",
                 "rescales", "kernel_launches"]


class FheLedger(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in LEDGER_FIELDS]


# (name, restype, argtypes)
SIGNATURES = [
    ("fhe_ctx_create", C.c_int, [C.POINTER(FheParams), vpp]),
    ("fhe_ctx_destroy", None, [vp]),
    ("fhe_last_error", C.c_char_p, [vp]),
    ("fhe_ctx_info", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int), u64p]),
    ("fhe_synchronize", C.c_int, [vp]),
    ("fhe_timer_start", C.c_int, [vp]),
    ("fhe_timer_stop", C.c_int, [vp, C.POINTER(C.c_float)]),
    ("fhe_prof_enable", C.c_int, [vp, C.c_int]),
    ("fhe_prof_get", C.c_int, [vp, C.c_char_p, C.POINTER(C.c_double), u64p]),
    ("fhe_prof_get_bytes", C.c_int, [vp, C.c_char_p, C.POINTER(C.c_double), u64p, C.POINTER(C.c_double)]),
    ("fhe_prof_reset", C.c_int, [vp]),
    ("fhe_profiler_range", C.c_int, [C.c_int]),
    ("fhe_bench_ntt", C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    ("fhe_ledger_get", C.c_int, [vp, C.POINTER(FheLedger)]),
    ("fhe_ledger_reset", C.c_int, [vp]),
    ("fhe_ledger_amounts", C.c_int, [vp, u64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("fhe_keygen", C.c_int, [vp, C.c_uint64]),
    ("fhe_gen_galois_keys", C.c_int, [vp, i64p, C.c_size_t]),
    ("fhe_galois_key_download", C.c_int, [vp, C.c_int64, u64p, C.c_size_t]),
    ("fhe_encode", C.c_int, [vp, dp, C.c_size_t, C.c_int, C.c_double, C.c_int, vpp]),
    ("fhe_encrypt", C.c_int, [vp, vp, C.c_uint64, vpp]),
    ("fhe_decrypt_decode", C.c_int, [vp, vp, dp, C.c_size_t]),
    ("fhe_ct_level", C.c_int, [vp]),
    ("fhe_ct_scale", C.c_double, [vp]),
    ("fhe_ct_download", C.c_int, [vp, vp, u64p, C.c_size_t]),
    ("fhe_ct_upload", C.c_int, [vp, u64p, C.c_int, C.c_double, vpp]),
    ("fhe_ct_upload_into", C.c_int, [vp, u64p, vp]),
    ("fhe_pt_download", C.c_int, [vp, vp, u64p, C.c_size_t]),
    ("fhe_pt_rows", C.c_int, [vp]),
    ("fhe_ct_free", None, [vp]),
    ("fhe_pt_free", None, [vp]),
    ("fhe_rotate", C.c_int, [vp, vp, C.c_int64, vpp]),
    ("fhe_rotate_hoisted", C.c_int, [vp, vp, i64p, C.c_size_t, vpp]),
    ("fhe_rotate_hoisted_batch", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, i64p, C.c_size_t, vpp]),
    ("fhe_rotate_hoisted_batch_into", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, i64p, C.c_size_t, vpp]),
    ("fhe_mul_plain", C.c_int, [vp, vp, vp, vpp]),
    ("fhe_add", C.c_int, [vp, vp, vp, vpp]),
    ("fhe_sub", C.c_int, [vp, vp, vp, vpp]),
    ("fhe_add_plain", C.c_int, [vp, vp, vp, vpp]),
    ("fhe_rescale", C.c_int, [vp, vp, vpp]),
    ("fhe_rotate_decomposed", C.c_int, [vp, vp, C.c_int64, C.c_int, vpp]),
    ("fhe_decompose", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, i64p, C.c_int]),
    ("fhe_conv_layer_create", C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_double, C.c_int, vpp]),
    ("fhe_conv_layer_free", None, [vp]),
    ("fhe_conv_layer_steps", C.c_int, [vp, C.c_int, i64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("fhe_conv2d", C.c_int, [vp, vp, vp, C.c_int, vpp]),
    ("fhe_conv2d_into", C.c_int, [vp, vp, vp, C.c_int, vp]),
    ("fhe_conv2d_batch", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, vp, C.c_int, vpp]),
    ("fhe_conv2d_batch_into", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, vp, C.c_int, C.POINTER(C.c_void_p)]),
    ("fhe_conv2d_batch_host", C.c_int, [vp, u64p, C.c_size_t, C.c_double, vp, C.c_int, C.c_size_t, u64p]),
    ("fhe_conv_layer_create_shards", C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_double, C.c_int,
                                               vpp]),
    ("fhe_conv_layer_shards", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("fhe_slot_sum_batch", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, C.c_uint64, vpp]),
    ("fhe_gen_relin_key", C.c_int, [vp]),
    ("fhe_add_scalar", C.c_int, [vp, vp, C.c_double, vpp]),
    ("fhe_mul_scalar", C.c_int, [vp, vp, C.c_double, vpp]),
    ("fhe_mul", C.c_int, [vp, vp, vp, vpp]),
    ("fhe_eval_chebyshev", C.c_int, [vp, vp, dp, C.c_size_t, C.c_double, C.c_int, vpp]),
    ("fhe_pool", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, C.c_int, C.c_int, vpp, C.POINTER(C.c_size_t),
                           i64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("fhe_subsample_stride2", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, C.c_int, C.c_int, vpp,
                                        C.POINTER(C.c_size_t), i64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("fhe_downsample", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, C.c_int, C.c_int, i64p, C.c_int, C.c_int,
                                 C.c_int, C.c_double, vpp, C.POINTER(C.c_size_t), i64p, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("fhe_linear_features", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, i64p, C.c_size_t, C.c_int, dp, dp,
                                      vpp]),
    ("fhe_conv_layer_create_packed", C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_double,
                                               C.c_int, C.c_size_t, i64p, C.c_int, C.c_int, vpp]),
    ("fhe_conv_layer_output_packing", C.c_int, [vp, C.POINTER(C.c_int)]),
    ("fhe_execute_schedule", C.c_int, [vp, vp, i64p, C.POINTER(C.c_int), C.c_size_t, C.c_int, vpp,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("fhe_linear", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, C.c_int, C.c_int, C.c_int, dp, dp, vpp]),
    ("fhe_conv2d_shards_into", C.c_int, [vp, C.POINTER(C.c_void_p), C.c_size_t, vp, C.POINTER(C.c_void_p)]),
    ("fhe_conv2d_batch_host_async", C.c_int, [vp, u64p, C.c_size_t, C.c_double, vp, C.c_int, C.c_size_t, u64p]),
    ("fhe_host_wait", C.c_int, [vp]),
]

EXPORTED = [s[0] for s in SIGNATURES]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libfheconv.so not built at {path}; run `python -m paper_2306_09189_b200.build` "
                          "(no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
