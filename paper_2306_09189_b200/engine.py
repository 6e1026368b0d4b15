"""Python host API over the C ABI (include/fheconv.h).

Mirrors the reference's evaluator surface (shardnn::Engine, reference
proj/include/shardnn/emu.hpp:132-183) and conv entry point (conv_plan,
proj/src/conv.cpp:266-271) so tests read like the reference's own tests:

    ctx = Context.from_config("cfg3")
    ctx.keygen(7)
    layer = ctx.conv_layer(c_in=16, c_out=16, m=32, kappa=3, weights=w)
    ctx.gen_galois_keys(layer.steps())
    ct = ctx.encrypt(ctx.encode(image_slots), seed=9000)
    out = ctx.conv2d(ct, layer, approach=2)       # ConvPlan::ShiftFirst
    slots = ctx.decrypt(out)

Every call goes to libfheconv.so on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Sequence

import numpy as np

from . import _lib

# BASELINE.json configs (CKKS parameters of cfg1..cfg5)
CONFIGS = {
    "cfg1": dict(log_n=13, q_bits=[60] + [40] * 4, p_bits=[60], log_scale=40),
    "cfg2": dict(log_n=14, q_bits=[50] * 8, p_bits=[60], log_scale=50),
    "cfg3": dict(log_n=15, q_bits=[60] + [50] * 12, p_bits=[60, 60], log_scale=50),
    "cfg4": dict(log_n=16, q_bits=[60] + [50] * 16, p_bits=[60, 60, 60], log_scale=50),
    "cfg5": dict(log_n=15, q_bits=[60] + [50] * 12, p_bits=[60, 60], log_scale=50),
}

_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib.load()
    return _L


class FheError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(FheError, ValueError):
    pass


def _u64(a):
    return a.ctypes.data_as(_lib.u64p)


class Plaintext:
    def __init__(self, ctx: "Context", h):
        self.ctx, self.h = ctx, h

    @property
    def rows(self) -> int:
        return lib().fhe_pt_rows(self.h)

    def residues(self) -> np.ndarray:
        out = np.zeros((self.rows, self.ctx.N), dtype=np.uint64)
        self.ctx._check(lib().fhe_pt_download(self.ctx.h, self.h, _u64(out), out.size))
        return out

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            lib().fhe_pt_free(self.h)
            self.h = None


class Ciphertext:
    def __init__(self, ctx: "Context", h):
        self.ctx, self.h = ctx, h

    @property
    def level(self) -> int:
        return lib().fhe_ct_level(self.h)

    @property
    def scale(self) -> float:
        return lib().fhe_ct_scale(self.h)

    def residues(self) -> np.ndarray:
        out = np.zeros((2, self.level + 1, self.ctx.N), dtype=np.uint64)
        self.ctx._check(lib().fhe_ct_download(self.ctx.h, self.h, _u64(out), out.size))
        return out

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            lib().fhe_ct_free(self.h)
            self.h = None


class ConvLayer:
    def __init__(self, ctx: "Context", h, c_in, c_out, m, kappa, level):
        self.ctx, self.h = ctx, h
        self.c_in, self.c_out, self.m, self.kappa, self.level = c_in, c_out, m, kappa, level

    def steps(self, approach: int = 0) -> list[int]:
        """Galois steps for `approach` (0: the union, so every schedule can run)."""
        buf = (C.c_int64 * 1024)()
        n = C.c_size_t(0)
        self.ctx._check(lib().fhe_conv_layer_steps(self.h, approach, buf, 1024, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def __del__(self):
        if getattr(self, "h", None) and self.ctx.h:
            lib().fhe_conv_layer_free(self.h)
            self.h = None


class Context:
    """One B200, one CUDA stream; owns keys and the cost ledger."""

    def __init__(self, log_n: int, q_bits: Sequence[int], p_bits: Sequence[int], log_scale: int, device: int = 0):
        self.log_n, self.N = log_n, 1 << log_n
        self.slots = self.N // 2
        self.q_bits, self.p_bits = list(q_bits), list(p_bits)
        qa = (C.c_int * len(q_bits))(*q_bits)
        pa = (C.c_int * len(p_bits))(*p_bits)
        self._keep = (qa, pa)
        p = _lib.FheParams(log_n, len(q_bits), qa, len(p_bits), pa, log_scale, device)
        h = C.c_void_p()
        rc = lib().fhe_ctx_create(C.byref(p), C.byref(h))
        if rc != 0:
            raise FheError(rc, f"fhe_ctx_create failed ({rc})")
        self.h = h.value
        nq, npp, dn = C.c_int(), C.c_int(), C.c_int()
        primes = (C.c_uint64 * (len(q_bits) + len(p_bits)))()
        lib().fhe_ctx_info(self.h, None, C.byref(nq), C.byref(npp), C.byref(dn), primes)
        self.L, self.K, self.dnum = nq.value, npp.value, dn.value
        self.primes = list(primes)
        self.scale = 2.0 ** log_scale
        self.max_level = self.L - 1

    @classmethod
    def from_config(cls, name: str, device: int = 0) -> "Context":
        return cls(device=device, **CONFIGS[name])

    def close(self):
        if getattr(self, "h", None):
            lib().fhe_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # ------------------------------------------------------------- helpers
    def _check(self, rc: int):
        if rc != 0:
            msg = lib().fhe_last_error(self.h).decode()
            if rc == _lib.FHE_E_INVALID:
                raise InvalidArgument(rc, msg)
            raise FheError(rc, msg)

    def _new(self, fn, *args, cls=Ciphertext):
        out = C.c_void_p()
        self._check(fn(self.h, *args, C.byref(out)))
        return cls(self, out.value)

    def synchronize(self):
        self._check(lib().fhe_synchronize(self.h))

    def timer_start(self):
        self._check(lib().fhe_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_float(0)
        self._check(lib().fhe_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def prof_enable(self, on: bool = True):
        self._check(lib().fhe_prof_enable(self.h, int(on)))

    def prof_reset(self):
        self._check(lib().fhe_prof_reset(self.h))

    def prof_get(self, cls: str) -> tuple[float, int]:
        ms, n, _ = self.prof_get_bytes(cls)
        return ms, n

    def prof_get_bytes(self, cls: str) -> tuple[float, int, float]:
        """(device ms, launches, algorithmic bytes) of a kernel class since prof_reset."""
        ms = C.c_double(0)
        n = C.c_uint64(0)
        b = C.c_double(0)
        self._check(lib().fhe_prof_get_bytes(self.h, cls.encode(), C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    # ---------------------------------------------------------------- keys
    def keygen(self, seed: int):
        self._check(lib().fhe_keygen(self.h, seed))

    def gen_galois_keys(self, steps: Iterable[int]):
        a = np.ascontiguousarray(list(steps), dtype=np.int64)
        self._check(lib().fhe_gen_galois_keys(self.h, a.ctypes.data_as(_lib.i64p), len(a)))

    def galois_key(self, step: int) -> np.ndarray:
        out = np.zeros((self.dnum, 2, self.L + self.K, self.N), dtype=np.uint64)
        self._check(lib().fhe_galois_key_download(self.h, step, _u64(out), out.size))
        return out

    # ---------------------------------------------------------------- data
    def encode(self, slots, level: int | None = None, scale: float | None = None,
               with_special: bool = False) -> Plaintext:
        z = np.ascontiguousarray(slots, dtype=np.float64)
        level = self.max_level if level is None else level
        scale = self.scale if scale is None else scale
        return self._new(lib().fhe_encode, z.ctypes.data_as(_lib.dp), len(z), level, scale, int(with_special),
                         cls=Plaintext)

    def encrypt(self, pt: Plaintext, seed: int) -> Ciphertext:
        return self._new(lib().fhe_encrypt, pt.h, seed)

    def decrypt(self, ct: Ciphertext, n: int | None = None) -> np.ndarray:
        n = self.slots if n is None else n
        out = np.zeros(n)
        self._check(lib().fhe_decrypt_decode(self.h, ct.h, out.ctypes.data_as(_lib.dp), n))
        return out

    def upload(self, residues: np.ndarray, level: int, scale: float | None = None) -> Ciphertext:
        r = np.ascontiguousarray(residues, dtype=np.uint64)
        assert r.size == 2 * (level + 1) * self.N
        return self._new(lib().fhe_ct_upload, _u64(r), level, self.scale if scale is None else scale)

    # ----------------------------------------------------------------- ops
    def rotate(self, ct: Ciphertext, k: int) -> Ciphertext:
        return self._new(lib().fhe_rotate, ct.h, k)

    def rotate_hoisted(self, ct: Ciphertext, ks: Sequence[int]) -> list[Ciphertext]:
        a = np.ascontiguousarray(list(ks), dtype=np.int64)
        outs = (C.c_void_p * max(1, len(a)))()
        self._check(lib().fhe_rotate_hoisted(self.h, ct.h, a.ctypes.data_as(_lib.i64p), len(a), outs))
        return [Ciphertext(self, outs[i]) for i in range(len(a))]

    rotate_many = rotate_hoisted  # reference name (emu.hpp:164)

    def rotate_hoisted_batch(self, cts: Sequence[Ciphertext], ks: Sequence[int]) -> list[list[Ciphertext]]:
        """fhe_rotate_hoisted_batch: [[rot_k(ct) for k in ks] for ct in cts], keys shared by the batch."""
        a = np.ascontiguousarray(list(ks), dtype=np.int64)
        ins = (C.c_void_p * max(1, len(cts)))(*[x.h for x in cts])
        outs = (C.c_void_p * max(1, len(cts) * len(a)))()
        self._check(lib().fhe_rotate_hoisted_batch(self.h, ins, len(cts), a.ctypes.data_as(_lib.i64p), len(a), outs))
        return [[Ciphertext(self, outs[i * len(a) + j]) for j in range(len(a))] for i in range(len(cts))]

    def rotate_hoisted_batch_into(self, cts: Sequence[Ciphertext], ks: Sequence[int], outs: Sequence[Ciphertext]):
        """fhe_rotate_hoisted_batch_into: outs[i * len(ks) + j] = rot_{ks[j]}(cts[i]) (preallocated)."""
        a = np.ascontiguousarray(list(ks), dtype=np.int64)
        ins = (C.c_void_p * max(1, len(cts)))(*[x.h for x in cts])
        o = (C.c_void_p * max(1, len(outs)))(*[x.h for x in outs])
        self._check(lib().fhe_rotate_hoisted_batch_into(self.h, ins, len(cts), a.ctypes.data_as(_lib.i64p), len(a), o))

    def rotate_decomposed(self, ct: Ciphertext, k: int, strategy: int) -> Ciphertext:
        return self._new(lib().fhe_rotate_decomposed, ct.h, k, strategy)

    def execute_schedule(self, ct: Ciphertext, amounts: Sequence[int], same_source: Sequence[int], strategy: int):
        """fhe_execute_schedule (reference plan_rotations + execute_schedule): returns
        (outputs, planned keyed rotations, groups, hoisted groups)."""
        n = len(amounts)
        a = np.ascontiguousarray(amounts, dtype=np.int64)
        ss = (C.c_int * max(1, n))(*[int(x) for x in same_source])
        outs = (C.c_void_p * max(1, n))()
        tot, g, gh = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        self._check(lib().fhe_execute_schedule(self.h, ct.h, a.ctypes.data_as(_lib.i64p), ss, n, strategy, outs,
                                               C.byref(tot), C.byref(g), C.byref(gh)))
        return [Ciphertext(self, outs[i]) for i in range(n)], tot.value, g.value, gh.value

    def mul_plain(self, ct: Ciphertext, pt: Plaintext) -> Ciphertext:
        return self._new(lib().fhe_mul_plain, ct.h, pt.h)

    def add(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        return self._new(lib().fhe_add, a.h, b.h)

    def sub(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        return self._new(lib().fhe_sub, a.h, b.h)

    def add_plain(self, ct: Ciphertext, pt: Plaintext) -> Ciphertext:
        return self._new(lib().fhe_add_plain, ct.h, pt.h)

    def rescale(self, ct: Ciphertext) -> Ciphertext:
        return self._new(lib().fhe_rescale, ct.h)

    # ---------------------------------------------------------------- conv
    @staticmethod
    def _bias(bias, c_out: int):
        """bias array (or None) for the C ABI; the reference's size check (conv.cpp:113-114)."""
        if bias is None or len(bias) == 0:
            return None, None
        b = np.ascontiguousarray(bias, dtype=np.float64)
        if b.size != c_out:
            raise ValueError("bias size does not match output channels")
        return b, b.ctypes.data_as(_lib.dp)

    def conv_layer(self, c_in: int, c_out: int, m: int, kappa: int, weights, level: int | None = None,
                   bias=None, output_scale: float = 1.0) -> ConvLayer:
        """fhe_conv_layer_create: conv_plan's layer (conv.hpp:66-68) with optional bias and output_scale."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        assert w.size == c_in * c_out * kappa * kappa
        level = self.max_level if level is None else level
        b, bp = self._bias(bias, c_out)
        out = C.c_void_p()
        self._check(lib().fhe_conv_layer_create(self.h, c_in, c_out, m, kappa, w.ctypes.data_as(_lib.dp), bp,
                                                float(output_scale), level, C.byref(out)))
        return ConvLayer(self, out.value, c_in, c_out, m, kappa, level)

    def conv_layer_shards(self, c_in: int, c_out: int, m: int, kappa: int, weights,
                          level: int | None = None, bias=None, output_scale: float = 1.0) -> ConvLayer:
        """fhe_conv_layer_create_shards: multi-shard image-mode layer (c_in m^2 = t * slots)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        assert w.size == c_in * c_out * kappa * kappa
        level = self.max_level if level is None else level
        b, bp = self._bias(bias, c_out)
        out = C.c_void_p()
        self._check(lib().fhe_conv_layer_create_shards(self.h, c_in, c_out, m, kappa, w.ctypes.data_as(_lib.dp),
                                                       bp, float(output_scale), level, C.byref(out)))
        ly = ConvLayer(self, out.value, c_in, c_out, m, kappa, level)
        t, no = C.c_int(0), C.c_int(0)
        self._check(lib().fhe_conv_layer_shards(ly.h, C.byref(t), C.byref(no)))
        ly.t, ly.n_out = t.value, no.value
        return ly

    def conv2d_shards(self, in_shards: Sequence[Ciphertext], layer: ConvLayer) -> list[Ciphertext]:
        """one or more images ([n_images * t] shards) -> [n_images * n_out] output shards."""
        n_img = len(in_shards) // layer.t
        assert n_img * layer.t == len(in_shards)
        outs = [self.encrypt(self.encode(np.zeros(8), level=layer.level - 1), 1) for _ in range(n_img * layer.n_out)]
        self.conv2d_shards_into(in_shards, layer, outs)
        return outs

    def conv2d_shards_into(self, in_shards: Sequence[Ciphertext], layer: ConvLayer, outs: Sequence[Ciphertext]):
        ins = (C.c_void_p * len(in_shards))(*[x.h for x in in_shards])
        o = (C.c_void_p * len(outs))(*[x.h for x in outs])
        self._check(lib().fhe_conv2d_shards_into(self.h, ins, len(in_shards) // layer.t, layer.h, o))

    def slot_sum_batch(self, cts: Sequence[Ciphertext], block: int) -> list[Ciphertext]:
        """fhe_slot_sum_batch: rotate-and-add block sums of every ciphertext (reference slot_sum)."""
        ins = (C.c_void_p * max(1, len(cts)))(*[x.h for x in cts])
        outs = (C.c_void_p * max(1, len(cts)))()
        self._check(lib().fhe_slot_sum_batch(self.h, ins, len(cts), block, outs))
        return [Ciphertext(self, outs[i]) for i in range(len(cts))]

    def pool(self, shards: Sequence[Ciphertext], c: int, m: int):
        """fhe_pool: 2x2 average pooling; returns (shards, tau, rep, d) like the reference's PackedImage."""
        return self._downsample(lib().fhe_pool, shards, c, m)

    def subsample_stride2(self, shards: Sequence[Ciphertext], c: int, m: int):
        """fhe_subsample_stride2 (reference subsample_stride2); returns (shards, tau, rep, d)."""
        return self._downsample(lib().fhe_subsample_stride2, shards, c, m)

    def _downsample(self, fn, shards, c, m):
        ins = (C.c_void_p * len(shards))(*[x.h for x in shards])
        outs = (C.c_void_p * len(shards))()
        n = C.c_size_t(0)
        tau = np.zeros(c, dtype=np.int64)
        rep, d = C.c_int(0), C.c_int(0)
        self._check(fn(self.h, ins, len(shards), c, m, outs, C.byref(n), tau.ctypes.data_as(_lib.i64p),
                       C.byref(rep), C.byref(d)))
        return [Ciphertext(self, outs[i]) for i in range(n.value)], tau, rep.value, d.value

    def downsample(self, shards: Sequence[Ciphertext], c: int, m: int, tau=None, rep: int = 1, d: int = 1,
                   window: bool = True, output_scale: float = 1.0):
        """fhe_downsample: pool (window) / stride-2 of any PackedImage; returns (shards, tau, rep, d, mode)."""
        ins = (C.c_void_p * len(shards))(*[x.h for x in shards])
        outs = (C.c_void_p * len(shards))()
        n = C.c_size_t(0)
        tau_out = np.zeros(c, dtype=np.int64)
        tin = None if tau is None else np.ascontiguousarray(tau, dtype=np.int64)
        rep_o, d_o, mode = C.c_int(0), C.c_int(0), C.c_int(0)
        self._check(lib().fhe_downsample(self.h, ins, len(shards), c, m,
                                         None if tin is None else tin.ctypes.data_as(_lib.i64p), rep, d,
                                         int(window), float(output_scale), outs, C.byref(n),
                                         tau_out.ctypes.data_as(_lib.i64p), C.byref(rep_o), C.byref(d_o),
                                         C.byref(mode)))
        return [Ciphertext(self, outs[i]) for i in range(n.value)], tau_out, rep_o.value, d_o.value, mode.value

    def gen_relin_key(self):
        self._check(lib().fhe_gen_relin_key(self.h))

    def add_scalar(self, ct: Ciphertext, k: float) -> Ciphertext:
        return self._new(lib().fhe_add_scalar, ct.h, float(k))

    def mul_scalar(self, ct: Ciphertext, k: float) -> Ciphertext:
        """ct * k in every slot, rescaled (one level, scale kept exactly)."""
        return self._new(lib().fhe_mul_scalar, ct.h, float(k))

    def mul(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        """fhe_mul: relinearised, rescaled ciphertext product (reference Engine::mul_ct)."""
        return self._new(lib().fhe_mul, a.h, b.h)

    def eval_chebyshev(self, ct: Ciphertext, coeffs, bound: float, prescaled: bool = False) -> Ciphertext:
        """fhe_eval_chebyshev: sum_k c_k T_k(x / bound) (reference eval_chebyshev)."""
        co = np.ascontiguousarray(coeffs, dtype=np.float64)
        return self._new(lib().fhe_eval_chebyshev, ct.h, co.ctypes.data_as(_lib.dp), co.size, bound, int(prescaled))

    def linear(self, shards: Sequence[Ciphertext], c: int, m: int, w, b) -> Ciphertext:
        """fhe_linear: W x + b over a packed image's features (reference linear())."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        ins = (C.c_void_p * len(shards))(*[x.h for x in shards])
        return self._new(lib().fhe_linear, ins, len(shards), c, m, len(b), w.ctypes.data_as(_lib.dp),
                         b.ctypes.data_as(_lib.dp))

    def linear_features(self, shards: Sequence[Ciphertext], features, w, b) -> Ciphertext:
        """fhe_linear_features: W x + b with an explicit slot -> feature map ([t][slots], -1 = none)."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        fm = np.ascontiguousarray(features, dtype=np.int64)
        assert fm.shape == (len(shards), self.slots)
        ins = (C.c_void_p * len(shards))(*[x.h for x in shards])
        return self._new(lib().fhe_linear_features, ins, len(shards), fm.ctypes.data_as(_lib.i64p),
                         w.size // len(b), len(b), w.ctypes.data_as(_lib.dp), b.ctypes.data_as(_lib.dp))

    def conv_layer_packed(self, c_in: int, c_out: int, m: int, kappa: int, weights, t: int = 1, tau=None,
                          rep: int = 1, d: int = 1, level: int | None = None, bias=None,
                          output_scale: float = 1.0) -> ConvLayer:
        """fhe_conv_layer_create_packed: image-mode layer over any PackedImage (tau, rep, d)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        assert w.size == c_in * c_out * kappa * kappa
        level = self.max_level if level is None else level
        b, bp = self._bias(bias, c_out)
        tv = None if tau is None else np.ascontiguousarray(tau, dtype=np.int64)
        out = C.c_void_p()
        self._check(lib().fhe_conv_layer_create_packed(self.h, c_in, c_out, m, kappa, w.ctypes.data_as(_lib.dp),
                                                       bp, float(output_scale), level, t,
                                                       None if tv is None else tv.ctypes.data_as(_lib.i64p),
                                                       rep, d, C.byref(out)))
        ly = ConvLayer(self, out.value, c_in, c_out, m, kappa, level)
        tt, no, dd = C.c_int(0), C.c_int(0), C.c_int(0)
        self._check(lib().fhe_conv_layer_shards(ly.h, C.byref(tt), C.byref(no)))
        self._check(lib().fhe_conv_layer_output_packing(ly.h, C.byref(dd)))
        ly.t, ly.n_out, ly.d_out = tt.value, no.value, dd.value
        return ly

    def conv2d(self, ct: Ciphertext, layer: ConvLayer, approach: int = 2) -> Ciphertext:
        return self._new(lib().fhe_conv2d, ct.h, layer.h, approach)

    def conv2d_into(self, ct: Ciphertext, layer: ConvLayer, approach: int, out: Ciphertext):
        self._check(lib().fhe_conv2d_into(self.h, ct.h, layer.h, approach, out.h))

    def conv2d_batch(self, cts: Sequence[Ciphertext], layer: ConvLayer, approach: int = 0) -> list[Ciphertext]:
        """n independent ciphertexts through one layer; keys and plaintexts are
        streamed once per batch (BSGS schedules)."""
        ins = (C.c_void_p * len(cts))(*[x.h for x in cts])
        outs = (C.c_void_p * len(cts))()
        self._check(lib().fhe_conv2d_batch(self.h, ins, len(cts), layer.h, approach, outs))
        return [Ciphertext(self, outs[i]) for i in range(len(cts))]

    def conv2d_batch_into(self, cts: Sequence[Ciphertext], layer: ConvLayer, approach: int,
                          outs: Sequence[Ciphertext]):
        ins = (C.c_void_p * len(cts))(*[x.h for x in cts])
        o = (C.c_void_p * len(outs))(*[x.h for x in outs])
        self._check(lib().fhe_conv2d_batch_into(self.h, ins, len(cts), layer.h, approach, o))

    def conv2d_batch_host(self, host_in, n: int, layer: ConvLayer, approach: int = 0, host_out=None,
                          chunk: int = 0, scale: float = 0.0, asynchronous: bool = False):
        """fhe_conv2d_batch_host: n host-resident ciphertexts (uint64 array [n, 2, level+1, N] or a raw
        pointer to one, e.g. a pinned torch tensor's data_ptr()) -> host_out ([n, 2, level, N]); uploads,
        convs and downloads of neighbouring chunks overlap."""
        lv = layer.level
        if host_out is None:
            host_out = np.empty((n, 2, lv, self.N), dtype=np.uint64)

        def ptr(x):
            if isinstance(x, int):
                return C.cast(x, _lib.u64p)
            assert x.dtype == np.uint64 and x.flags["C_CONTIGUOUS"]
            return x.ctypes.data_as(_lib.u64p)
        fn = lib().fhe_conv2d_batch_host_async if asynchronous else lib().fhe_conv2d_batch_host
        self._check(fn(self.h, ptr(host_in), n, scale, layer.h, approach, chunk, ptr(host_out)))
        return host_out

    def host_wait(self):
        """fhe_host_wait: completes every conv2d_batch_host(..., asynchronous=True)."""
        self._check(lib().fhe_host_wait(self.h))

    # -------------------------------------------------------------- ledger
    def ledger(self) -> dict:
        lg = _lib.FheLedger()
        self._check(lib().fhe_ledger_get(self.h, C.byref(lg)))
        return {f: getattr(lg, f) for f in _lib.LEDGER_FIELDS}

    def ledger_reset(self):
        self._check(lib().fhe_ledger_reset(self.h))

    def rotation_amounts(self) -> list[int]:
        buf = (C.c_uint64 * 4096)()
        n = C.c_size_t(0)
        self._check(lib().fhe_ledger_amounts(self.h, buf, 4096, C.byref(n)))
        return [buf[i] for i in range(min(n.value, 4096))]


def decompose(strategy: int, n: int, s: int) -> list[int]:
    """reference rot.cpp:21-46 (0 = positive, 1 = signed)."""
    buf = (C.c_int64 * 64)()
    k = lib().fhe_decompose(strategy, n, s, buf, 64)
    if k < 0:
        raise InvalidArgument(k, "amount must satisfy 0 <= n < s")
    return [buf[i] for i in range(k)]
