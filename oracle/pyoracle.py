"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module. It binds:
  * oracle/_build/liboracle.so  — this repo's C restatement (emu_ref.c,
    ckks_ref.c, mt19937.c): the checker for the product's residues;
  * oracle/_ref/libshardnn_ref.so — the UNMODIFIED reference sources compiled
    where they lie (plus ref_shim.cpp); present only where it was built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import math

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libshardnn_ref.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
lp = C.POINTER(C.c_long)


def build():
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.ck_create.restype = C.c_void_p
        L.ck_create.argtypes = [C.c_int, C.c_int, ip, C.c_int, ip, C.c_int]
        L.ck_destroy.argtypes = [C.c_void_p]
        for name in ("ck_prime", "ck_root"):
            getattr(L, name).restype = C.c_uint64
            getattr(L, name).argtypes = [C.c_void_p, C.c_int]
        L.ck_dnum.argtypes = [C.c_void_p]
        L.ck_dnum_at.argtypes = [C.c_void_p, C.c_int]
        L.ck_scale.restype = C.c_double
        L.ck_scale.argtypes = [C.c_void_p]
        L.ck_mulmod.restype = C.c_uint64
        L.ck_mulmod.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ck_is_prime.argtypes = [C.c_uint64]
        L.ck_galois_elt.restype = C.c_uint64
        L.ck_galois_elt.argtypes = [C.c_void_p, C.c_long]
        L.ck_automorph_ntt.argtypes = [C.c_void_p, u64p, u64p, C.c_uint64]
        L.ck_automorph_coef.argtypes = [C.c_void_p, C.c_int, u64p, u64p, C.c_uint64]
        L.ck_ntt_fwd.argtypes = [C.c_void_p, C.c_int, u64p]
        L.ck_ntt_inv.argtypes = [C.c_void_p, C.c_int, u64p]
        L.ck_encode.argtypes = [C.c_void_p, dp, C.c_size_t, C.c_double, i64p]
        L.ck_decode.argtypes = [C.c_void_p, dp, C.c_double, dp]
        L.ck_encode_plain.argtypes = [C.c_void_p, dp, C.c_size_t, C.c_double, C.c_int, C.c_int, u64p]
        L.ck_prng.restype = C.c_uint64
        L.ck_prng.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ck_keygen.argtypes = [C.c_void_p, C.c_uint64]
        L.ck_secret_coef.argtypes = [C.c_void_p, i64p]
        L.ck_galois_key.argtypes = [C.c_void_p, C.c_uint64, u64p]
        L.ck_encrypt.argtypes = [C.c_void_p, u64p, C.c_int, C.c_uint64, u64p]
        L.ck_decrypt_coef.argtypes = [C.c_void_p, u64p, C.c_int, dp]
        L.ck_decrypt_decode.argtypes = [C.c_void_p, u64p, C.c_int, C.c_double, dp]
        for name in ("ck_add", "ck_mul_plain", "ck_add_plain"):
            getattr(L, name).argtypes = [C.c_void_p, u64p, u64p, C.c_int, u64p]
        L.ck_rescale.argtypes = [C.c_void_p, u64p, C.c_int, u64p]
        L.ck_modup.argtypes = [C.c_void_p, u64p, C.c_int, u64p]
        L.ck_inner_product.argtypes = [C.c_void_p, u64p, C.c_int, u64p, C.c_uint64, u64p, u64p]
        L.ck_moddown.argtypes = [C.c_void_p, u64p, C.c_int, u64p]
        L.ck_rotate.argtypes = [C.c_void_p, u64p, C.c_int, C.c_long, u64p]
        L.ck_mul_ct.argtypes = [C.c_void_p, u64p, u64p, C.c_int, u64p]
        L.ck_rotate_hoisted.argtypes = [C.c_void_p, u64p, C.c_int, lp, C.c_int, u64p]
        L.ck_conv.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp,
                              C.c_int, u64p, dp]
        L.ck_conv_shards.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp,
                                     u64p, dp]
        L.ck_conv_packed.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp,
                                     lp, C.c_int, C.c_int, u64p, dp]
        L.ck_conv_channel.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp, u64p, dp]
        L.ck_lintrans.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, lp, u64p, u64p]
        L.ck_lintrans_src.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), lp, u64p,
                                      u64p]
        L.emu_make_inputs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                      C.c_int, dp, dp]
        L.emu_rotate.argtypes = [dp, dp, C.c_size_t, C.c_long]
        L.emu_fused_plain.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, dp, C.c_int,
                                      C.c_long, C.c_long, C.c_double, dp]
        L.emu_conv_slots.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, dp, dp,
                                     C.c_int, dp]
        L.emu_oracle_conv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, dp]
        L.emu_fused_plain_ms.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, dp, C.c_int, C.c_int,
                                         C.c_int, C.c_long, C.c_long, C.c_double, dp]
        L.emu_conv_shards_slots.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, dp, dp, dp]
        L.emu_conv_channel_slots.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, dp, dp, dp]
        L.emu_decompose.argtypes = [C.c_int, C.c_uint64, C.c_uint64, lp, C.c_int]
        L.emu_min_lengths.argtypes = [C.c_uint64, C.c_uint64, u64p]
        _lib = L
    return _lib


_CHEB_FN = C.CFUNCTYPE(C.c_double, C.c_double)


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(REF_SO)
        R.ref_make_inputs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                      C.c_int, dp, dp]
        R.ref_conv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, C.c_uint64, dp,
                               dp, u64p, ip]
        R.ref_conv_biased.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, C.c_uint64, dp,
                                      C.c_double, dp, C.c_int, u64p]
        R.ref_oracle_conv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, dp]
        R.ref_decompose.argtypes = [C.c_int, C.c_uint64, C.c_uint64, lp, C.c_int]
        R.ref_min_lengths.argtypes = [C.c_uint64, C.c_uint64, u64p]
        R.ref_plan_rotations.restype = C.c_long
        R.ref_plan_rotations.argtypes = [lp, ip, C.c_int, C.c_uint64, C.c_int, lp, ip, ip, ip]
        R.ref_time_conv.restype = C.c_double
        R.ref_time_conv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, C.c_uint64,
                                    C.c_int, C.c_int]
        R.ref_linear.argtypes = [C.c_int, C.c_int, dp, C.c_int, dp, dp, C.c_uint64, dp, u64p]
        R.ref_pool.argtypes = [C.c_int, C.c_int, dp, C.c_uint64, dp, C.c_int, u64p, u64p, u64p]
        R.ref_write_network.argtypes = [C.c_int, C.c_char_p, C.c_uint64]
        R.ref_run_network.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_int, C.c_int, dp, dp, C.c_int,
                                      C.POINTER(C.c_int64), dp, C.POINTER(C.c_int64), u64p, C.c_char_p, C.c_uint64]
        R.ref_pool_conv.argtypes = [C.c_int, C.c_int, dp, C.c_uint64, C.c_int, C.c_int, dp, dp, C.c_int, u64p]
        R.ref_downsample.argtypes = [C.c_int, C.c_int, dp, C.c_uint64, C.c_int, C.c_double, dp, C.c_int, u64p, u64p,
                                     u64p]
        R.ref_slot_sum.argtypes = [dp, C.c_uint64, C.c_uint64, dp]
        R.ref_eval_chebyshev.argtypes = [dp, C.c_uint64, C.c_int, dp, C.c_uint64, C.c_double, C.c_int, dp,
                                         C.POINTER(C.c_int64), u64p, C.c_char_p, C.c_uint64]
        R.ref_cheb_interpolate.argtypes = [_CHEB_FN, C.c_uint64, C.c_double, dp]
        R.ref_time_rotations.restype = C.c_double
        R.ref_time_rotations.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, u64p]
        _ref = R
    return _ref


# ---------------------------------------------------------------- emulator

def make_inputs(c, m, kappa, c_out, seed_img, seed_filt, weight_kind=0, use_ref=False):
    img = np.zeros(c * m * m)
    filt = np.zeros(c * c_out * kappa * kappa)
    fn = ref().ref_make_inputs if use_ref else lib().emu_make_inputs
    rc = fn(c, m, kappa, c_out, seed_img, seed_filt, weight_kind, _ptr(img, dp), _ptr(filt, dp))
    assert rc in (0, None)
    return img, filt


def emu_conv_slots(c, m, kappa, c_out, s, img, filt, plan):
    out = np.zeros(s)
    img = np.ascontiguousarray(img, dtype=np.float64)
    filt = np.ascontiguousarray(filt, dtype=np.float64)
    rc = lib().emu_conv_slots(c, m, kappa, c_out, s, _ptr(img, dp), _ptr(filt, dp), plan, _ptr(out, dp))
    assert rc == 0
    return out


def emu_conv_shards_slots(c, m, kappa, c_out, s, img, filt):
    """conv_image_shards slots ([n_out][s]) of a multi-shard image (t = c m^2 / s shards)."""
    z = s // (m * m)
    n_out = 1 if c_out <= z else c_out // z
    out = np.zeros(n_out * s)
    rc = lib().emu_conv_shards_slots(c, m, kappa, c_out, s, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp),
                                     _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), _ptr(out, dp))
    assert rc == n_out, rc
    return out.reshape(n_out, s)


def emu_conv_channel_slots(c, m, kappa, c_out, s, img, filt):
    """conv_channel_shards slots ([c_out * m^2 / s][s]) of a channel-shard image (m^2 > s)."""
    n = c_out * (m * m // s)
    out = np.zeros(n * s)
    rc = lib().emu_conv_channel_slots(c, m, kappa, c_out, s, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp),
                                      _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), _ptr(out, dp))
    assert rc == n, rc
    return out.reshape(n, s)


def ref_conv_channel(c, m, kappa, c_out, img, filt, s):
    """the reference's convolve() on a channel-shard image: conv_channel_shards slots."""
    n = c_out * (m * m // s)
    out_slots = np.zeros(n * s)
    out_img = np.zeros(c_out * m * m)
    ledger = np.zeros(9, dtype=np.uint64)
    drop = C.c_int(0)
    rc = ref().ref_conv(c, m, kappa, c_out, _ptr(np.ascontiguousarray(img), dp), _ptr(np.ascontiguousarray(filt), dp),
                        0, s, _ptr(out_slots, dp), _ptr(out_img, dp), _ptr(ledger, u64p), C.byref(drop))
    assert rc == 0
    return out_slots.reshape(n, s), out_img, ledger, drop.value


def ref_linear(c, m, img, w, b, s):
    """the reference's linear() (dense.cpp:71-75) on pack(img, s): output slots, ledger, shard count."""
    out = np.zeros(s)
    ledger = np.zeros(9, dtype=np.uint64)
    t = ref().ref_linear(c, m, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp), len(b),
                         _ptr(np.ascontiguousarray(w, dtype=np.float64), dp),
                         _ptr(np.ascontiguousarray(b, dtype=np.float64), dp), s, _ptr(out, dp), _ptr(ledger, u64p))
    assert t > 0, t
    return out, ledger, t


def ref_pool(c, m, img, s):
    """the reference's pool() of pack(img, s): (shard slots [n][s], meta [m, c, d, rep, mode, n], tau, ledger)."""
    out = np.zeros(16 * s)
    meta = np.zeros(6, dtype=np.uint64)
    tau = np.zeros(c, dtype=np.uint64)
    ledger = np.zeros(9, dtype=np.uint64)
    n = ref().ref_pool(c, m, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp), s, _ptr(out, dp), 16,
                       _ptr(meta, u64p), _ptr(tau, u64p), _ptr(ledger, u64p))
    assert n > 0, n
    return out[: n * s].reshape(n, s), meta, tau, ledger


def ref_downsample(c, m, img, s, window=True, output_scale=1.0, cap=64):
    """the reference's pool() (window) / subsample_stride2() of pack(img, s):
    (shard slots [n][s], meta [m, c, d, rep, mode, n, rows_per_shard], tau, ledger)."""
    out = np.zeros(cap * s)
    meta = np.zeros(7, dtype=np.uint64)
    tau = np.zeros(c, dtype=np.uint64)
    ledger = np.zeros(9, dtype=np.uint64)
    n = ref().ref_downsample(c, m, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp), s, int(window),
                             float(output_scale), _ptr(out, dp), cap, _ptr(meta, u64p), _ptr(tau, u64p),
                             _ptr(ledger, u64p))
    assert n > 0, n
    return out[: n * s].reshape(n, s), meta, tau, ledger


def ref_write_network(which, directory, side=16):
    """the reference's test networks (tests/test_net.cpp, tiny_net.hpp) written as JSON + fixtures
    with the reference's own io.cpp savers."""
    assert ref().ref_write_network(which, str(directory).encode(), side) == 0


def ref_run_network(json_path, input_path, shard_size=0, initial_level=0, auto_boot=-1):
    """the reference's run_network (net.cpp:112-257) on a JSON network: dict with logits,
    oracle_logits, per-layer info [level_before, level_after, depth, bootstrapped], errors,
    ledger totals; raises RuntimeError with the reference's message."""
    cap = 64
    lg, ol = np.zeros(cap), np.zeros(cap)
    info = np.zeros(4 * 32, dtype=np.int64)
    err = np.zeros(32)
    meta = np.zeros(2, dtype=np.int64)
    tot = np.zeros(8, dtype=np.uint64)
    msg = C.create_string_buffer(512)
    rc = ref().ref_run_network(str(json_path).encode(), str(input_path).encode(), shard_size, initial_level,
                               auto_boot, _ptr(lg, dp), _ptr(ol, dp), cap,
                               info.ctypes.data_as(C.POINTER(C.c_int64)), _ptr(err, dp),
                               meta.ctypes.data_as(C.POINTER(C.c_int64)), _ptr(tot, u64p), msg, 512)
    if rc != 0:
        raise RuntimeError(msg.value.decode())
    nl, no = int(meta[0]), int(meta[1])
    return dict(logits=lg[:no].copy(), oracle_logits=ol[:no].copy(), info=info[:4 * nl].reshape(nl, 4).copy(),
                errors=err[:nl].copy(), totals=tot.copy())


def ref_pool_conv(c, m, img, s, kappa, c_out, filt, cap=16):
    """the reference's convolve(pool(pack(img, s)), k): (conv shard slots [n][s], meta [m, c, d, rep, mode, n])."""
    out = np.zeros(cap * s)
    meta = np.zeros(6, dtype=np.uint64)
    n = ref().ref_pool_conv(c, m, _ptr(np.ascontiguousarray(img, dtype=np.float64), dp), s, kappa, c_out,
                            _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), _ptr(out, dp), cap,
                            _ptr(meta, u64p))
    assert n > 0, n
    return out[: n * s].reshape(n, s), meta


def ref_slot_sum(vec, block):
    vec = np.ascontiguousarray(vec, dtype=np.float64)
    out = np.zeros(vec.size)
    assert ref().ref_slot_sum(_ptr(vec, dp), vec.size, block, _ptr(out, dp)) == 0
    return out


def ref_eval_chebyshev(x, level, coeffs, bound, prescaled):
    """the reference's eval_chebyshev (act.cpp:151-162) on slots x at `level`:
    (slots, output level, max depth, ledger) or raises RuntimeError with its text."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    co = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros(x.size)
    meta = (C.c_int64 * 2)()
    ledger = np.zeros(9, dtype=np.uint64)
    err = C.create_string_buffer(256)
    rc = ref().ref_eval_chebyshev(_ptr(x, dp), x.size, level, _ptr(co, dp), co.size, bound, int(prescaled),
                                  _ptr(out, dp), meta, _ptr(ledger, u64p), err, 256)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return out, meta[0], meta[1], ledger


def ref_cheb_interpolate(f, n, bound):
    """the reference's cheb_interpolate (act.cpp:90-113)."""
    co = np.zeros(n + 1)
    cb = _CHEB_FN(f)
    assert ref().ref_cheb_interpolate(cb, n, bound, _ptr(co, dp)) == 0
    return co


def cheb_interpolate(f, n, bound):
    """restatement of act.cpp:90-113: Chebyshev interpolant through the n+1
    Chebyshev nodes (same loop order and rounding as the reference)."""
    if bound <= 0.0:
        raise ValueError("bound must be positive")
    pts = n + 1
    y = [f(bound * math.cos(math.pi * (2.0 * j + 1.0) / (2.0 * pts))) for j in range(pts)]
    co = []
    for k in range(pts):
        acc = 0.0
        for j in range(pts):
            acc += y[j] * math.cos(math.pi * k * (2.0 * j + 1.0) / (2.0 * pts))
        co.append(2.0 * acc / pts)
    co[0] /= 2.0
    return np.array(co)


def cheb_eval(coeffs, bound, x):
    """Clenshaw evaluation (act.cpp:115-125), vectorised over x."""
    t = np.asarray(x, dtype=np.float64) / bound
    b1 = np.zeros_like(t)
    b2 = np.zeros_like(t)
    for k in range(len(coeffs) - 1, 0, -1):
        b1, b2 = 2.0 * t * b1 - b2 + coeffs[k], b1
    return t * b1 - b2 + coeffs[0]


def emu_oracle_conv(c, m, kappa, c_out, img, filt):
    out = np.zeros(c_out * m * m)
    lib().emu_oracle_conv(c, m, kappa, c_out, _ptr(np.ascontiguousarray(img), dp),
                          _ptr(np.ascontiguousarray(filt), dp), _ptr(out, dp))
    return out


def emu_fused_plain(c, m, kappa, c_out, s, filt, r, kk, ll):
    out = np.zeros(s)
    ne = lib().emu_fused_plain(c, m, kappa, c_out, s, _ptr(np.ascontiguousarray(filt), dp), r, kk, ll,
                               1.0, _ptr(out, dp))
    return out if ne else None


def emu_decompose(strategy, n, s):
    buf = (C.c_long * 64)()
    k = lib().emu_decompose(strategy, n, s, buf, 64)
    assert k >= 0
    return [buf[i] for i in range(k)]


def emu_min_lengths(n_max, cap):
    out = np.zeros(n_max + 1, dtype=np.uint64)
    assert lib().emu_min_lengths(n_max, cap, _ptr(out, u64p)) == 0
    return out


def ref_conv(c, m, kappa, c_out, img, filt, plan, s):
    out_slots = np.zeros(s)
    out_img = np.zeros(c_out * m * m)
    ledger = np.zeros(9, dtype=np.uint64)
    drop = C.c_int(0)
    rc = ref().ref_conv(c, m, kappa, c_out, _ptr(np.ascontiguousarray(img), dp),
                        _ptr(np.ascontiguousarray(filt), dp), plan, s, _ptr(out_slots, dp),
                        _ptr(out_img, dp), _ptr(ledger, u64p), C.byref(drop))
    assert rc == 0
    return out_slots, out_img, ledger, drop.value


def ref_conv_shards(c, m, kappa, c_out, img, filt, s):
    """the reference's convolve() on a multi-shard image: conv_image_shards slots [n_out][s]."""
    z = s // (m * m)
    n_out = 1 if c_out <= z else c_out // z
    out_slots = np.zeros(n_out * s)
    out_img = np.zeros(c_out * m * m)
    ledger = np.zeros(9, dtype=np.uint64)
    drop = C.c_int(0)
    rc = ref().ref_conv(c, m, kappa, c_out, _ptr(np.ascontiguousarray(img), dp), _ptr(np.ascontiguousarray(filt), dp),
                        0, s, _ptr(out_slots, dp), _ptr(out_img, dp), _ptr(ledger, u64p), C.byref(drop))
    assert rc == 0
    return out_slots.reshape(n_out, s), out_img, ledger, drop.value


def ref_conv_biased(c, m, kappa, c_out, img, filt, plan, s, bias, output_scale, cap=64):
    """conv_plan / convolve with bias and output_scale (conv.hpp:46-68): output slots [n_out][s]."""
    out = np.zeros(cap * s)
    ledger = np.zeros(9, dtype=np.uint64)
    n = ref().ref_conv_biased(c, m, kappa, c_out, _ptr(np.ascontiguousarray(img), dp),
                              _ptr(np.ascontiguousarray(filt), dp), plan, s,
                              _ptr(np.ascontiguousarray(bias, dtype=np.float64), dp), float(output_scale),
                              _ptr(out, dp), cap, _ptr(ledger, u64p))
    assert n > 0
    return out[: n * s].reshape(n, s), ledger


# ---------------------------------------------------------------- CKKS model

class CKKS:
    """Thin owner of a ck_ctx (the CPU golden model)."""

    def __init__(self, logN, qbits, pbits, logscale):
        L = lib()
        self.logN, self.N = logN, 1 << logN
        self.qbits, self.pbits = list(qbits), list(pbits)
        self.L, self.K = len(qbits), len(pbits)
        qa = (C.c_int * self.L)(*qbits)
        pa = (C.c_int * self.K)(*pbits)
        self.h = L.ck_create(logN, self.L, qa, self.K, pa, logscale)
        assert self.h
        self.np = self.L + self.K
        self.primes = [L.ck_prime(self.h, i) for i in range(self.np)]
        self.dnum = L.ck_dnum(self.h)
        self.scale = L.ck_scale(self.h)

    def __del__(self):
        try:
            lib().ck_destroy(self.h)
        except Exception:
            pass

    def dnum_at(self, level):
        return lib().ck_dnum_at(self.h, level)

    def keygen(self, seed):
        lib().ck_keygen(self.h, seed)

    def secret(self):
        s = np.zeros(self.N, dtype=np.int64)
        lib().ck_secret_coef(self.h, _ptr(s, i64p))
        return s

    def galois(self, k):
        return lib().ck_galois_elt(self.h, k)

    def galois_key(self, g):
        key = np.zeros((self.dnum, 2, self.np, self.N), dtype=np.uint64)
        lib().ck_galois_key(self.h, g, _ptr(key, u64p))
        return key

    def ntt(self, idx, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        (lib().ck_ntt_inv if inverse else lib().ck_ntt_fwd)(self.h, idx, _ptr(a, u64p))
        return a

    def encode_coef(self, z, scale):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.zeros(self.N, dtype=np.int64)
        rc = lib().ck_encode(self.h, _ptr(z, dp), len(z), scale, _ptr(out, i64p))
        assert rc == 0
        return out

    def decode(self, coef, scale):
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        z = np.zeros(self.N // 2)
        lib().ck_decode(self.h, _ptr(coef, dp), scale, _ptr(z, dp))
        return z

    def encode(self, z, scale, level, with_p=False):
        z = np.ascontiguousarray(z, dtype=np.float64)
        rows = level + 1 + (self.K if with_p else 0)
        out = np.zeros((rows, self.N), dtype=np.uint64)
        rc = lib().ck_encode_plain(self.h, _ptr(z, dp), len(z), scale, level, int(with_p), _ptr(out, u64p))
        assert rc == 0
        return out

    def encrypt(self, pt, level, seed):
        ct = np.zeros((2, level + 1, self.N), dtype=np.uint64)
        lib().ck_encrypt(self.h, _ptr(np.ascontiguousarray(pt), u64p), level, seed, _ptr(ct, u64p))
        return ct

    def decrypt(self, ct, level, scale):
        z = np.zeros(self.N // 2)
        lib().ck_decrypt_decode(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, scale, _ptr(z, dp))
        return z

    def decrypt_coef(self, ct, level):
        z = np.zeros(self.N)
        lib().ck_decrypt_coef(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, _ptr(z, dp))
        return z

    def _binop(self, fn, a, b, level):
        out = np.zeros((2, level + 1, self.N), dtype=np.uint64)
        fn(self.h, _ptr(np.ascontiguousarray(a), u64p), _ptr(np.ascontiguousarray(b), u64p), level,
           _ptr(out, u64p))
        return out

    def add(self, a, b, level):
        return self._binop(lib().ck_add, a, b, level)

    def mul_plain(self, ct, pt, level):
        return self._binop(lib().ck_mul_plain, ct, pt, level)

    def add_plain(self, ct, pt, level):
        return self._binop(lib().ck_add_plain, ct, pt, level)

    def rescale(self, ct, level):
        out = np.zeros((2, level, self.N), dtype=np.uint64)
        lib().ck_rescale(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, _ptr(out, u64p))
        return out

    def modup(self, c1, level):
        out = np.zeros((self.dnum_at(level), level + 1 + self.K, self.N), dtype=np.uint64)
        lib().ck_modup(self.h, _ptr(np.ascontiguousarray(c1), u64p), level, _ptr(out, u64p))
        return out

    def moddown(self, acc, level):
        out = np.zeros((level + 1, self.N), dtype=np.uint64)
        lib().ck_moddown(self.h, _ptr(np.ascontiguousarray(acc), u64p), level, _ptr(out, u64p))
        return out

    def rotate(self, ct, level, k):
        out = np.zeros((2, level + 1, self.N), dtype=np.uint64)
        lib().ck_rotate(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, k, _ptr(out, u64p))
        return out

    def mul_ct(self, a, b, level):
        """relinearised, rescaled product (ck_mul_ct): [2][level+1][N] x2 -> [2][level][N]."""
        out = np.zeros((2, level, self.N), dtype=np.uint64)
        lib().ck_mul_ct(self.h, _ptr(np.ascontiguousarray(a[:, : level + 1]), u64p),
                        _ptr(np.ascontiguousarray(b[:, : level + 1]), u64p), level, _ptr(out, u64p))
        return out

    def eval_chebyshev(self, ct, level, scale, coeffs, bound, prescaled):
        """Chebyshev series on a ciphertext: the reference's split (act.cpp:49-82, 151-162)
        with the scale targeting of fheconv.cu's ChebEval, op for op, so the residues
        are comparable bit for bit. Returns (ct, level, scale)."""
        primes = self.primes

        def const(k, lv, sc):
            # the constant polynomial round(k * sc): its NTT rows are the constant itself
            v = float(np.rint(k * sc))
            assert abs(v) < 9.2e18
            iv = int(v)
            return np.stack([np.full(self.N, iv % int(primes[i]), dtype=np.uint64) for i in range(lv + 1)])

        def drop(v, lv):
            c, l0, sc = v
            if l0 < lv:
                raise RuntimeError("insufficient level for activation: bootstrap required")
            return (np.ascontiguousarray(c[:, : lv + 1]), lv, sc)

        def add(a, b):
            assert a[1] == b[1]
            return (self.add(a[0], b[0], a[1]), a[1], a[2])

        def add_scalar(v, k):
            return (self.add_plain(v[0], const(k, v[1], v[2]), v[1]), v[1], v[2])

        def mul_scalar(v, k, lv, sc):
            c, _, vs = drop(v, lv + 1)
            pr = self.mul_plain(c, const(k, lv + 1, sc * float(primes[lv + 1]) / vs), lv + 1)
            return (self.rescale(pr, lv + 1), lv, sc)

        def mul(a, b):
            lv = a[1]
            assert b[1] == lv
            return (self.mul_ct(a[0], b[0], lv), lv - 1, a[2] * b[2] / float(primes[lv]))

        def floor_pow2(d):
            p = 1
            while p * 2 <= d:
                p *= 2
            return p

        basis = []

        def of_degree(p2):
            return basis[p2.bit_length() - 1]

        def series(co, lv, sc):
            d = len(co) - 1
            if d <= 2:
                acc = mul_scalar(of_degree(1), co[1], lv, sc)
                if d == 2:
                    acc = add(acc, mul_scalar(of_degree(2), co[2], lv, sc))
                return add_scalar(acc, co[0])
            p = floor_pow2(d)
            if p == d:
                top = mul_scalar(of_degree(p), co[d], lv, sc)
                return add(top, series(co[:-1], lv, sc))
            q = [0.0] * (d - p + 1)
            r = list(co[: p + 1])
            for a in range(1, d - p + 1):
                q[a] = 2.0 * co[p + a]
                r[p - a] -= co[p + a]
            tp = drop(of_degree(p), lv + 1)
            qv = series(q, lv + 1, sc * float(primes[lv + 1]) / tp[2])
            prod = mul(qv, tp)
            return add((prod[0], prod[1], sc), series(r, lv, sc))

        co = [float(v) for v in coeffs]
        d = len(co) - 1
        needed = d.bit_length() + (0 if prescaled else 1)
        if level < needed:
            raise RuntimeError("insufficient level for activation: bootstrap required")
        out_level = level - needed
        t = (np.ascontiguousarray(ct), level, scale)
        if not prescaled:
            t = mul_scalar(t, 1.0 / bound, level - 1, scale)
        if d == 0:  # the reference's fresh encode (act.cpp:158)
            pt = const(co[0], level, scale)
            return (np.stack([pt, np.zeros_like(pt)]), level, scale)
        basis.append(t)
        p = 2
        while p <= floor_pow2(d):
            half = basis[-1]
            sq = mul(half, half)
            basis.append(add_scalar(add(sq, sq), -1.0))
            p *= 2
        return series(co, out_level, scale)

    def rotate_hoisted(self, ct, level, ks):
        out = np.zeros((len(ks), 2, level + 1, self.N), dtype=np.uint64)
        ka = (C.c_long * len(ks))(*ks)
        lib().ck_rotate_hoisted(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, ka, len(ks),
                                _ptr(out, u64p))
        return out

    def conv(self, ct, level, c, m, kappa, c_out, filt, plan):
        out = np.zeros((2, level, self.N), dtype=np.uint64)
        sc = C.c_double(0)
        rc = lib().ck_conv(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, c, m, kappa, c_out,
                           _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), plan, _ptr(out, u64p),
                           C.byref(sc))
        assert rc == 0
        return out, sc.value

    def conv_shards(self, cts, level, c, m, kappa, c_out, filt):
        """multi-shard image-mode conv: cts [t][2][level+1][N] -> [n_out][2][level][N]."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        t = cts.shape[0]
        z = (self.N // 2) // (m * m)
        n_out = 1 if c_out <= z else c_out // z
        out = np.zeros((n_out, 2, level, self.N), dtype=np.uint64)
        sc = C.c_double(0)
        rc = lib().ck_conv_shards(self.h, _ptr(cts, u64p), t, level, c, m, kappa, c_out,
                                  _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), _ptr(out, u64p),
                                  C.byref(sc))
        assert rc == n_out, rc
        return out, sc.value

    def lintrans(self, ct, level, amounts, slot_vectors):
        """Rescale(ModDown(sum_b pt_b * rot_{amounts[b]}(ct))), pt_b = slot_vectors[b] encoded over
        Q_level u P at scale q_level."""
        pts = np.stack([self.encode(v, float(self.primes[level]), level, with_p=True) for v in slot_vectors])
        a = (C.c_long * len(amounts))(*amounts)
        out = np.zeros((2, level, self.N), dtype=np.uint64)
        lib().ck_lintrans(self.h, _ptr(np.ascontiguousarray(ct), u64p), level, len(amounts), a,
                          _ptr(np.ascontiguousarray(pts), u64p), _ptr(out, u64p))
        return out

    def lintrans_src(self, cts, level, terms):
        """Rescale(ModDown(sum pt * rot_amount(cts[src]))) over terms (src, amount, slot vector), all
        accumulated in the QP basis before one ModDown + rescale."""
        cts = np.ascontiguousarray(np.stack(cts), dtype=np.uint64)
        pts = np.stack([self.encode(v, float(self.primes[level]), level, with_p=True) for _, _, v in terms])
        src = (C.c_int * len(terms))(*[t[0] for t in terms])
        a = (C.c_long * len(terms))(*[t[1] for t in terms])
        out = np.zeros((2, level, self.N), dtype=np.uint64)
        lib().ck_lintrans_src(self.h, _ptr(cts, u64p), cts.shape[0], level, len(terms), src, a,
                              _ptr(np.ascontiguousarray(pts), u64p), _ptr(out, u64p))
        return out

    def conv_packed(self, cts, level, c, m, kappa, c_out, filt, tau, rep, d):
        """image-mode conv over a PackedImage (tau, rep, d): cts [t][2][level+1][N] -> [n_out][2][level][N]."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        t = cts.shape[0]
        z = (self.N // 2) // (m * m)
        n_out = 1 if c_out <= z else c_out // z
        out = np.zeros((n_out, 2, level, self.N), dtype=np.uint64)
        sc = C.c_double(0)
        tv = (C.c_long * c)(*[int(x) for x in tau])
        rc = lib().ck_conv_packed(self.h, _ptr(cts, u64p), t, level, c, m, kappa, c_out,
                                  _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), tv, rep, d, _ptr(out, u64p),
                                  C.byref(sc))
        assert rc == n_out, rc
        return out, sc.value

    def conv_channel(self, cts, level, c, m, kappa, c_out, filt):
        """channel-shard conv: cts [c * pc][2][level+1][N] -> [c_out * pc][2][level][N]."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        pc = m * m // (self.N // 2)
        out = np.zeros((c_out * pc, 2, level, self.N), dtype=np.uint64)
        sc = C.c_double(0)
        rc = lib().ck_conv_channel(self.h, _ptr(cts, u64p), level, c, m, kappa, c_out,
                                   _ptr(np.ascontiguousarray(filt, dtype=np.float64), dp), _ptr(out, u64p),
                                   C.byref(sc))
        assert rc == c_out * pc, rc
        return out, sc.value


# ------------------------------------------------------------------ pooling restatement
class NumpyOps:
    """slot-vector backend of downsample_restated (the reference's arithmetic, no cryptography)."""

    @staticmethod
    def lintrans(srcs, terms):
        return sum(v * np.roll(srcs[j], -a) for j, a, v in terms)

    @staticmethod
    def rotate(x, k):
        return np.roll(x, -k)

    @staticmethod
    def add(a, b):
        return a + b


class CkksOps:
    """golden CKKS backend: items are (residues, level); lintrans = ck_lintrans_src (all terms in
    the QP basis, one ModDown + rescale), rotate = ck_rotate, add = ck_add."""

    def __init__(self, ck):
        self.ck = ck

    def lintrans(self, srcs, terms):
        lv = srcs[0][1]
        return self.ck.lintrans_src([x for x, _ in srcs], lv, terms), lv - 1

    def rotate(self, x, k):
        return self.ck.rotate(x[0], x[1], k), x[1]

    def add(self, a, b):
        return self.ck.add(a[0], b[0], a[1]), a[1]


def downsample_restated(ops, xs, c, m, s, window=True, oscale=1.0, d_in=1, tau_in=None, rep_in=1):
    """pool() / subsample_stride2() (pool.cpp:10-306) restated in the rotation-of-mask form the
    GPU runs (rot_k(x * mask) = rot_k(mask) * rot_k(x)): window (image: pool.cpp:22-30; channel
    shards with the next shard's spill masks: :34-72), horizontal (:76-86) and vertical (:90-129)
    stages as plaintext-weighted sums of rotations, then consolidation (:167-273) and channel
    duplication (:276-289). Returns (shards, tau, rep, d, mode)."""
    block = m * m
    image = block <= s
    t = len(xs)
    tau0 = list(range(c)) if tau_in is None else list(tau_in)
    pc, rows = (1, 0) if image else (block // s, s // m)
    rot = lambda v, k: np.roll(v, -k)
    X = list(xs)
    if window:
        if image:
            terms = []
            for kk, ll in ((0, 0), (0, 1), (1, 0), (1, 1)):
                v = np.zeros(s)
                for b in range(s // block):
                    for i in range(m - kk):
                        v[b * block + i * m: b * block + i * m + (m - ll)] = 0.25
                terms.append((0, kk * m + ll, v))
            X = [ops.lintrans([x], terms) for x in X]
        else:
            full, last = [], []
            for kk, ll in ((0, 0), (0, 1), (1, 0), (1, 1)):
                inm, spm = np.zeros(s), np.zeros(s)
                for rr in range(rows):
                    (inm if rr + kk < rows else spm)[rr * m: rr * m + (m - ll)] = 0.25
                if inm.any():
                    full.append((0, kk * m + ll, inm))
                    last.append((0, kk * m + ll, inm))
                if spm.any():
                    full.append((1, kk * m + ll, spm))
            X = [ops.lintrans([X[u], X[u + 1]], full) if (u % pc) + 1 < pc else ops.lintrans([X[u]], last)
                 for u in range(t)]
    live = [u for u in range(t) if image or rows != 1 or ((u % pc) * rows) % 2 == 0]
    hterms = []
    for i in range(m // 2):
        mk = np.zeros(s)
        mk[2 * i::m] = 1.0
        hterms.append((0, i, rot(mk, i)))
    R, vblock = (m, block) if image else (rows, s)
    vterms = []
    if R == 1:
        mv = np.zeros(s)
        mv[: m // 2] = oscale
        vterms.append((0, 0, mv))
    for j in range(R // 2):
        mv = np.zeros(s)
        for b in range(s // vblock):
            mv[b * vblock + 2 * j * m: b * vblock + 2 * j * m + m // 2] = oscale
        vterms.append((0, 3 * j * m // 2, rot(mv, 3 * j * m // 2)))
    V = [None] * t
    for u in live:
        V[u] = ops.lintrans([ops.lintrans([X[u]], hterms)], vterms)
    mn = m // 2
    bn = mn * mn
    tau, rep, d, mode, dup, stride = [0] * c, 1, 1, 0, 1, 0
    res = []
    if image:
        z = c * d_in // t
        if t == 1:
            res, tau, rep, d, dup, stride = [V[0]], tau0, 4 * rep_in, 4 * d_in, 4, bn
        elif t == 2:
            res = [ops.add(V[0], ops.rotate(V[1], -2 * bn))]
            tau = [tau0[(j % 2) * z + j // 2] for j in range(c)]
            rep, d, dup, stride = 2, 2, 2, bn
        else:
            for w in range(t // 4):
                acc = V[4 * w]
                for q in range(1, 4):
                    acc = ops.add(acc, ops.rotate(V[4 * w + q], -q * bn))
                res.append(acc)
                for g in range(4 * z):
                    tau[w * 4 * z + g] = tau0[(4 * w + g % 4) * z + g // 4]
    else:
        for w in range((t + 3) // 4):
            acc = None
            for q in range(4):
                if 4 * w + q >= t or V[4 * w + q] is None:
                    continue
                term = V[4 * w + q] if q == 0 else ops.rotate(V[4 * w + q], -q * (s // 4))
                acc = term if acc is None else ops.add(acc, term)
            res.append(acc)
        tau = list(range(c))
        if bn > s:
            mode = 1
        else:
            valid = c * bn
            d = s // valid if valid < s else 1
            if d > 1:
                dup, stride = d, valid
    if dup > 1:
        base = res[0]
        out = base
        for e in range(1, dup):
            out = ops.add(out, ops.rotate(base, -e * stride))
        res = [out]
    return res, np.array(tau), rep, d, mode


def downsample_steps(c, m, s, window=True):
    """the Galois steps downsample_restated / fhe_downsample rotate by (nonzero, reduced mod s)."""
    block, mn = m * m, m // 2
    image = block <= s
    rows = 0 if image else s // m
    st = set()
    if window:
        st |= {1, m, m + 1}
    st |= set(range(1, m // 2))
    R = m if image else rows
    st |= {3 * j * m // 2 for j in range(R // 2)}
    bn = mn * mn
    if image:
        st |= {-q * bn for q in range(1, 4)}
    else:
        st |= {-q * (s // 4) for q in range(1, 4)}
        if bn <= s and c * bn < s:
            st |= {-e * c * bn for e in range(1, s // (c * bn))}
    return sorted({k % s for k in st if k % s})
