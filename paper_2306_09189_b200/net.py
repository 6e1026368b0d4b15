"""JSON network runner on real ciphertexts (reference net.cpp:51-257).

`load_network` reads the reference's JSON network description (net.cpp:51-110:
shard_size, initial_level, seed, layers of type conv / pool / gelu / linear /
pool_linear with fixture files resolved next to the JSON) and `run_network`
executes it on RNS-CKKS ciphertexts through this library's C ABI — every
layer's arithmetic runs in libfheconv's sm_100a kernels — beside the
reference's plaintext mirror (net.cpp:140-223: the same polynomial activation
evaluated in the clear), reporting per-layer levels, errors, ledger deltas and
the logit residuals exactly like RunReport (net.hpp:57-80).

Differences forced by real cryptography (network runner):
  * the shard size is the context's slot count (N/2): packing is a layout
    choice and the reference's outputs do not depend on it; a spec's
    shard_size is recorded but the image is packed (and duplicated) at N/2;
  * there is no bootstrapping (out of scope), so the run starts at
    min(initial_level, ctx.max_level) and a layer that needs more levels than
    are left raises the reference's "level underflow at layer ..." error, as
    net.cpp:160-164 does with bootstrap.auto = false.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .engine import Ciphertext, Context
from .fixtures import ChebPoly, FilterTensor, ImageTensor, LinearWeights, load_filter, load_linear, load_poly

LAYER_TYPES = ("conv", "pool", "gelu", "linear", "pool_linear")


# ----------------------------------------------------------------- specs
@dataclass
class LayerSpec:
    """net.hpp:16-33"""
    type: str
    name: str = ""
    filter: Optional[FilterTensor] = None
    bias: np.ndarray = field(default_factory=lambda: np.zeros(0))
    bn_scale: Optional[np.ndarray] = None
    bn_bias: Optional[np.ndarray] = None
    stride: int = 1
    degree: int = 59
    bound: float = 10.0
    poly: Optional[ChebPoly] = None
    weights: Optional[LinearWeights] = None


@dataclass
class NetworkSpec:
    """net.hpp:40-47"""
    shard_size: int = 4096
    initial_level: int = 30
    seed: int = 0
    bootstrap_auto: bool = True
    layers: list = field(default_factory=list)


def load_network(path: str) -> NetworkSpec:
    """net.cpp:51-110: the JSON format, fixture paths relative to the JSON file."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise RuntimeError("cannot open " + path) from None
    d = os.path.dirname(path)
    res = lambda p: os.path.join(d, p)
    spec = NetworkSpec(shard_size=int(j.get("shard_size", 4096)), initial_level=int(j.get("initial_level", 30)),
                       seed=int(j.get("seed", 0)), bootstrap_auto=bool(j.get("bootstrap", {}).get("auto", True)))
    for lj in j["layers"]:
        t = lj["type"]
        ly = LayerSpec(type=t, name=lj.get("name", t))
        if t == "conv":
            ly.filter, ly.bias = load_filter(res(lj["filter"]))
            ly.stride = int(lj.get("stride", 1))
            if "bn_scale" in lj:
                ly.bn_scale = np.asarray(lj["bn_scale"], dtype=np.float64)
                ly.bn_bias = np.asarray(lj["bn_bias"], dtype=np.float64)
        elif t == "pool":
            pass
        elif t == "gelu":
            ly.degree = int(lj.get("degree", 59))
            ly.bound = float(lj.get("bound", 10.0))
            if "poly" in lj:
                ly.poly = load_poly(res(lj["poly"]))
                if "bound" in lj and ly.poly.bound != ly.bound:
                    raise RuntimeError("layer bound does not match its polynomial fixture")
                ly.bound, ly.degree = ly.poly.bound, ly.poly.degree
        elif t in ("linear", "pool_linear"):
            ly.weights = load_linear(res(lj["weights"]))
        else:
            raise RuntimeError("unknown layer type: " + t)
        spec.layers.append(ly)
    return spec


# ------------------------------------------------------- host math (planning)
def oracle_gelu(x: float) -> float:
    """oracle.cpp:78-81"""
    return x * 0.5 * (1.0 + math.erf(x / math.sqrt(2.0)))


def cheb_interpolate(f, n: int, bound: float) -> ChebPoly:
    """act.cpp:103-125: interpolation at the n + 1 Chebyshev nodes of [-bound, bound]."""
    if bound <= 0.0:
        raise ValueError("bound must be positive")
    pts = n + 1
    y = [f(bound * math.cos(math.pi * (2.0 * j + 1.0) / (2.0 * pts))) for j in range(pts)]
    co = np.zeros(pts)
    for k in range(pts):
        acc = 0.0
        for j in range(pts):
            acc += y[j] * math.cos(math.pi * k * (2.0 * j + 1.0) / (2.0 * pts))
        co[k] = 2.0 * acc / pts
    co[0] /= 2.0
    return ChebPoly(co, bound)


def cheb_eval(poly: ChebPoly, x):
    """act.cpp:127-137 (Clenshaw), elementwise"""
    t = np.asarray(x, dtype=np.float64) / poly.bound
    b1 = np.zeros_like(t)
    b2 = np.zeros_like(t)
    for k in range(poly.degree, 0, -1):
        b1, b2 = 2.0 * t * b1 - b2 + poly.coeffs[k], b1
    return t * b1 - b2 + poly.coeffs[0]


def chebyshev_required_level(degree: int) -> int:
    """act.cpp: bit length of the degree"""
    bits = 0
    while (1 << bits) <= degree:
        bits += 1
    return bits


def fold_bn(k: FilterTensor, bias: np.ndarray, scale: np.ndarray, shift: np.ndarray):
    """dense.cpp:5-21"""
    if scale.size != k.c_out or shift.size != k.c_out:
        raise ValueError("batch norm size does not match output channels")
    if bias.size and bias.size != k.c_out:
        raise ValueError("bias size does not match output channels")
    w = k.weights.reshape(k.c_in, k.c_out, k.kappa, k.kappa) * scale[None, :, None, None]
    b = scale * (bias if bias.size else np.zeros(k.c_out)) + shift
    return FilterTensor(k.c_in, k.c_out, k.kappa, w.reshape(-1)), b


def oracle_conv(t: ImageTensor, k: FilterTensor, stride: int = 1) -> ImageTensor:
    """oracle.cpp:7-31: same-padded cross-correlation with centred taps"""
    if k.c_in != t.c:
        raise ValueError("input channel mismatch")
    h = k.kappa // 2
    x = np.pad(t.data.reshape(t.c, t.m, t.m), ((0, 0), (h, h), (h, h)))
    w = k.weights.reshape(k.c_in, k.c_out, k.kappa, k.kappa)
    out = np.zeros((k.c_out, t.m, t.m))
    for r in range(k.kappa):
        for s in range(k.kappa):
            out += np.einsum("fg,fij->gij", w[:, :, r, s], x[:, r:r + t.m, s:s + t.m])
    if stride == 2:
        out = out[:, ::2, ::2]
    return ImageTensor(k.c_out, out.shape[1], out)


def oracle_avgpool2x2(t: ImageTensor) -> ImageTensor:
    x = t.data.reshape(t.c, t.m, t.m)
    p = 0.25 * (x[:, 0::2, 0::2] + x[:, 1::2, 0::2] + x[:, 0::2, 1::2] + x[:, 1::2, 1::2])
    return ImageTensor(t.c, t.m // 2, p)


def required_level(ly: LayerSpec, prescaled: bool) -> int:
    """net.cpp:33-43"""
    if ly.type == "conv":
        return 3 if ly.stride == 2 else 1
    if ly.type == "pool":
        return 3
    if ly.type == "gelu":
        return chebyshev_required_level(ly.degree) + (0 if prescaled else 1)
    return 2


# --------------------------------------------------------- packed ciphertexts
@dataclass
class PackedCiphertexts:
    """PackedImage (pack.hpp) whose shards are ciphertexts in HBM"""
    shards: list
    m: int
    c: int
    tau: np.ndarray
    rep: int = 1
    d: int = 1
    mode: int = 0  # 0 image shards, 1 channel shards

    def min_level(self) -> int:
        return min(s.level for s in self.shards)

    def block_channel(self, g: int) -> int:
        return int(self.tau[(g // self.rep) % self.c])


def pack_slots(t: ImageTensor, s: int):
    """pack.cpp:7-49 -> (shard slot vectors, d, mode)"""
    block = t.m * t.m
    if block <= s:
        d = s // (block * t.c) if block * t.c < s else 1
        flat = np.tile(t.data, d)
        return list(flat.reshape(-1, s)), d, 0
    return list(t.data.reshape(-1, s)), 1, 1


def slot_feature_map(p: PackedCiphertexts, s: int) -> np.ndarray:
    """pack.cpp:109-129: feature held by every slot, -1 for non-primary replicas / padding"""
    block = p.m * p.m
    fm = -np.ones((len(p.shards), s), dtype=np.int64)
    if p.mode == 0:
        per = s // block
        for g in range(len(p.shards) * per):
            if not (g < p.c * p.rep and g % p.rep == 0):
                continue
            ch = p.block_channel(g)
            fm[g // per, (g % per) * block:(g % per + 1) * block] = ch * block + np.arange(block)
    else:
        pc = block // s
        for ch in range(p.c):
            for u in range(pc):
                fm[ch * pc + u] = ch * block + u * s + np.arange(s)
    return fm


def unpack_slots(p: PackedCiphertexts, slots: Sequence[np.ndarray], s: int) -> np.ndarray:
    """pack.cpp:84-107"""
    fm = slot_feature_map(p, s)
    out = np.zeros(p.c * p.m * p.m)
    for u, v in enumerate(slots):
        sel = fm[u] >= 0
        out[fm[u][sel]] = v[sel]
    return out


def downsample_steps(c: int, m: int, s: int, rep: int, d: int, t: int, mode: int, window: bool) -> set:
    """rotations of pool / subsample_stride2 as fhe_downsample runs them (pool.cpp:10-306)"""
    block, mn = m * m, m // 2
    bn = mn * mn
    st = set(range(1, m // 2))
    if window:
        st |= {1, m, m + 1}
    R = m if mode == 0 else s // m
    st |= {3 * j * m // 2 for j in range(R // 2)}
    if mode == 0:
        st |= {-q * bn for q in range(1, 4)}
    else:
        st |= {-q * (s // 4) for q in range(1, 4)}
        if bn <= s and c * bn < s:
            st |= {-e * c * bn for e in range(1, s // (c * bn))}
    return {k % s for k in st if k % s}


# --------------------------------------------------------------- reports
LEDGER_KEYS = ("rotations", "hoisted_rotations", "hoist_groups", "ct_pt_mults", "ct_ct_mults", "adds",
               "bootstraps", "key_switches")


@dataclass
class LayerReport:
    name: str
    type: str
    bootstrapped: bool = False
    level_before: int = 0
    level_after: int = 0
    depth_consumed: int = 0
    max_abs_err: float = 0.0
    ops: dict = field(default_factory=dict)


@dataclass
class RunReport:
    layers: list = field(default_factory=list)
    logits: np.ndarray = field(default_factory=lambda: np.zeros(0))
    oracle_logits: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residual_mean: float = 0.0
    residual_std: float = 0.0
    residual_max: float = 0.0
    totals: dict = field(default_factory=dict)
    bootstrap_layers: list = field(default_factory=list)
    shard_size: int = 0
    initial_level: int = 0

    def to_text(self) -> str:
        """RunReport::to_text (net.cpp:259-283)"""
        out = ["layer                 type         lvl before->after  boot  max|err|"]
        for i, l in enumerate(self.layers):
            out.append(f"{i:<2} {l.name:<18} {l.type:<12} {l.level_before:3d} -> {l.level_after:<3d}        "
                       f"{'yes' if l.bootstrapped else 'no':<5} {l.max_abs_err:.9e}")
        out.append("logits: " + " ".join(f"{v:.9e}" for v in self.logits))
        out.append("oracle: " + " ".join(f"{v:.9e}" for v in self.oracle_logits))
        out.append(f"residual mean {self.residual_mean:.9e} std {self.residual_std:.9e} max {self.residual_max:.9e}")
        t = self.totals
        out.append(f"ledger: rot {t.get('rotations', 0)} hoisted {t.get('hoisted_rotations', 0)} ct_pt "
                   f"{t.get('ct_pt_mults', 0)} ct_ct {t.get('ct_ct_mults', 0)} add {t.get('adds', 0)} boot 0 "
                   f"key_switches {t.get('key_switches', 0)}")
        return "\n".join(out) + "\n"


# ------------------------------------------------------------------ runner
class _Keys:
    def __init__(self, ctx: Context):
        self.ctx, self.have, self.relin = ctx, set(), False

    def need(self, steps):
        s = self.ctx.slots
        new = sorted({k % s for k in steps if k % s} - self.have)
        if new:
            self.ctx.gen_galois_keys(new)
            self.have |= set(new)

    def need_relin(self):
        if not self.relin:
            self.ctx.gen_relin_key()
            self.relin = True


def _ledger_delta(a: dict, b: dict) -> dict:
    return {k: int(b.get(k, 0)) - int(a.get(k, 0)) for k in b}


def _plan(spec: NetworkSpec):
    """activation bounds fold into the closest preceding conv / pool (net.cpp:128-146)"""
    n = len(spec.layers)
    fold, pre, polys = [1.0] * n, [False] * n, [None] * n
    for i, ly in enumerate(spec.layers):
        if ly.type != "gelu":
            continue
        polys[i] = ly.poly if ly.poly is not None else cheb_interpolate(oracle_gelu, ly.degree, ly.bound)
        if i > 0 and spec.layers[i - 1].type in ("conv", "pool"):
            fold[i - 1] = 1.0 / ly.bound
            pre[i] = True
    return fold, pre, polys


def mirror_network(spec: NetworkSpec, x: ImageTensor):
    """the plaintext mirror of run_network (net.cpp:166-223): per layer (mirror tensor, carried
    scale) and the oracle logits. Host-side check data, never on the encrypted path."""
    fold, pre, polys = _plan(spec)
    mirror, carried, states = ImageTensor(x.c, x.m, x.data.copy()), 1.0, []
    for i, ly in enumerate(spec.layers):
        if ly.type == "conv":
            k, bias = ly.filter, ly.bias
            if ly.bn_scale is not None:
                k, bias = fold_bn(k, bias, ly.bn_scale, ly.bn_bias)
            mirror = oracle_conv(mirror, k, ly.stride)
            if bias.size:
                mirror = ImageTensor(mirror.c, mirror.m,
                                     (mirror.data.reshape(mirror.c, -1) + bias[:, None]).reshape(-1))
            carried *= fold[i]
        elif ly.type == "pool":
            mirror = oracle_avgpool2x2(mirror)
            carried *= fold[i]
        elif ly.type == "gelu":
            mirror = ImageTensor(mirror.c, mirror.m, cheb_eval(polys[i], mirror.data))
            carried = 1.0
        else:
            w = ly.weights
            xin = mirror.data if ly.type == "linear" else mirror.data.reshape(mirror.c, -1).mean(axis=1)
            if xin.size != w.in_features:
                raise ValueError("in_features mismatch")
            return states, w.w.reshape(w.out_features, -1) @ xin + w.b
        states.append((mirror, carried))
    raise ValueError("network must end with a linear layer")


def run_network(ctx: Context, spec: NetworkSpec, x: ImageTensor, enc_seed: int = 9000,
                check_layers: bool = True, cache: Optional[dict] = None) -> RunReport:
    """run_network (net.cpp:112-257) on ciphertexts. The context must hold a
    secret key (ctx.keygen); Galois and relinearisation keys are generated on
    demand. check_layers decrypts every intermediate map to report its error
    against the mirror (the reference always does; the timed path skips it). `cache`
    (a dict owned by the caller) keeps the encoded conv layers between runs of the
    same network, the serving case: layer plaintexts are encoded once."""
    if not spec.layers:
        raise ValueError("network has no layers")
    s = ctx.slots
    fold, pre, polys = _plan(spec)
    states, oracle_logits = mirror_network(spec, x)
    keys = _Keys(ctx)
    rep = RunReport(shard_size=s, initial_level=min(spec.initial_level, ctx.max_level))
    lv0 = rep.initial_level
    slots, d, mode = pack_slots(x, s)
    cts = [ctx.encrypt(ctx.encode(v, level=lv0), enc_seed + u) for u, v in enumerate(slots)]
    p = PackedCiphertexts(cts, x.m, x.c, np.arange(x.c), 1, d, mode)
    terminal = False
    logits_ct = None
    for i, ly in enumerate(spec.layers):
        if terminal:
            raise ValueError("linear layers must come last")
        lr = LayerReport(name=ly.name or ly.type, type=ly.type, level_before=p.min_level())
        need = required_level(ly, pre[i])
        if lr.level_before < need:
            raise RuntimeError(f"level underflow at layer {i} ({lr.name}): need {need}, have {lr.level_before}")
        before = ctx.ledger()
        if ly.type == "conv":
            k, bias = ly.filter, ly.bias
            if ly.bn_scale is not None:
                k, bias = fold_bn(k, bias, ly.bn_scale, ly.bn_bias)
            p = _conv(ctx, keys, p, k, bias, fold[i], cache, i)
            if ly.stride == 2:
                p = _downsample(ctx, keys, p, False, 1.0)
        elif ly.type == "pool":
            p = _downsample(ctx, keys, p, True, fold[i])
        elif ly.type == "gelu":
            keys.need_relin()
            poly = polys[i]
            p = PackedCiphertexts([ctx.eval_chebyshev(sh, poly.coeffs, poly.bound, pre[i]) for sh in p.shards],
                                  p.m, p.c, p.tau, p.rep, p.d, p.mode)
        else:
            w = ly.weights
            feats = slot_feature_map(p, s)
            if ly.type == "linear":
                if w.in_features != p.c * p.m * p.m:
                    raise ValueError("in_features does not match the packed feature count")
                wf = w.w
            else:
                if w.in_features != p.c:
                    raise ValueError("pool-linear expects one input feature per channel")
                block = p.m * p.m
                wf = np.repeat(w.w.reshape(w.out_features, p.c), block, axis=1).reshape(-1) / block
            if w.out_features > s:
                raise ValueError("out_features exceeds the shard size")
            keys.need(1 << j for j in range(int(math.log2(s))))
            logits_ct = ctx.linear_features(p.shards, feats, wf, w.b)
            rep.oracle_logits = oracle_logits
            terminal = True
        lr.ops = _ledger_delta(before, ctx.ledger())
        if terminal:
            lr.level_after = logits_ct.level
            rep.logits = ctx.decrypt(logits_ct)[: ly.weights.out_features]
            lr.max_abs_err = float(np.abs(rep.logits - rep.oracle_logits).max())
        else:
            lr.level_after = p.min_level()
            if check_layers:
                mirror, carried = states[i]
                dec = unpack_slots(p, [ctx.decrypt(sh) for sh in p.shards], s)
                lr.max_abs_err = float(np.abs(dec - mirror.data * carried).max())
        lr.depth_consumed = lr.level_before - lr.level_after
        rep.layers.append(lr)
    if not terminal:
        raise ValueError("network must end with a linear layer")
    rep.totals = ctx.ledger()
    r = rep.logits - rep.oracle_logits
    rep.residual_mean = float(r.mean())
    rep.residual_std = float(np.sqrt(((r - r.mean()) ** 2).mean()))
    rep.residual_max = float(np.abs(r).max())
    return rep


def _conv(ctx: Context, keys: _Keys, p: PackedCiphertexts, k: FilterTensor, bias: np.ndarray,
          scale: float, cache: Optional[dict] = None, idx: int = -1) -> PackedCiphertexts:
    """convolve (conv.cpp:364-371) with the folded output scale and the bias (conv.cpp:87-94, :344):
    both are properties of the libfheconv layer (fhe_conv_layer_create_*: the scale folded into the
    fused plaintexts, the bias added in the conv epilogue)"""
    if k.c_in != p.c:
        raise ValueError("filter input channels do not match image")
    if bias.size and bias.size != k.c_out:
        raise ValueError("bias size does not match output channels")
    b = bias if bias.size else None
    lv = p.min_level()
    ck = (idx, p.mode, len(p.shards), tuple(int(v) for v in p.tau), p.rep, p.d, lv, scale)
    layer = cache.get(ck) if cache is not None else None
    if p.mode == 1:
        if layer is None:
            layer = ctx.conv_layer_shards(k.c_in, k.c_out, p.m, k.kappa, k.weights, level=lv, bias=b,
                                          output_scale=scale)
        if cache is not None:
            cache[ck] = layer
        keys.need(layer.steps())
        outs = ctx.conv2d_shards(p.shards, layer)
        return PackedCiphertexts(outs, p.m, k.c_out, np.arange(k.c_out), 1, 1, 1)
    if layer is None:
        layer = ctx.conv_layer_packed(k.c_in, k.c_out, p.m, k.kappa, k.weights, t=len(p.shards), tau=p.tau,
                                      rep=p.rep, d=p.d, level=lv, bias=b, output_scale=scale)
    if cache is not None:
        cache[ck] = layer
    keys.need(layer.steps())
    outs = ctx.conv2d_shards(p.shards, layer)
    return PackedCiphertexts(outs, p.m, k.c_out, np.arange(k.c_out), 1, layer.d_out, 0)


def _downsample(ctx: Context, keys: _Keys, p: PackedCiphertexts, window: bool, scale: float) -> PackedCiphertexts:
    s = ctx.slots
    keys.need(downsample_steps(p.c, p.m, s, p.rep, p.d, len(p.shards), p.mode, window))
    outs, tau, rep, d, mode = ctx.downsample(p.shards, p.c, p.m, tau=p.tau, rep=p.rep, d=p.d, window=window,
                                             output_scale=scale)
    return PackedCiphertexts(outs, p.m // 2, p.c, tau, rep, d, mode)


def bench_network(ctx: Context, spec: NetworkSpec, x: ImageTensor, repetitions: int) -> dict:
    """bench_network (net.cpp:285-310): repeats the run, aggregates ledger counters by
    layer type and checks they are identical across runs."""
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    first, same = None, True
    for _ in range(repetitions):
        ctx.ledger_reset()
        r = run_network(ctx, spec, x, check_layers=False)
        # the reference's counters (CostLedger::Snapshot); GPU work counters such as kernel
        # launches also count the keys generated on the first run
        sig = [{k: l.ops.get(k, 0) for k in LEDGER_KEYS} for l in r.layers]
        if first is None:
            first = (r, sig)
        else:
            same = same and sig == first[1]
    per_type: dict = {}
    for l in first[0].layers:
        agg = per_type.setdefault(l.type, {})
        for k2, v in l.ops.items():
            agg[k2] = agg.get(k2, 0) + v
    return {"per_type": per_type, "repetitions": repetitions, "deterministic": same}
