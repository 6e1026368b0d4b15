"""Generates tests/golden/golden.npz from the UNMODIFIED reference.

Run in the container that has /root/reference (the GPU box does not):
    make -C oracle && python tests/golden/make_golden.py

Every value comes from the reference's own code compiled where it lies
(oracle/_ref/libshardnn_ref.so built by oracle/Makefile; ref_shim.cpp only
adapts calling conventions): inputs from its test helpers
(tests/helpers.hpp:13-27), conv outputs and ledgers from conv_plan /
convolve (conv.cpp:254-371), decompositions from rot.cpp:21-129.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

# name: (c, m, kappa, c_out, seed_img, seed_filt, weight_kind, shard size s)
CONV_CASES = {
    "cfg1": (4, 32, 3, 4, 1000, 2000, 0, 4096),
    "cfg3": (16, 32, 3, 16, 1001, 2001, 0, 16384),
    "cfg4": (8, 64, 5, 8, 1002, 2002, 2, 32768),
    "small_c4m4k3": (4, 4, 3, 4, 39, 139, 0, 64),
    "small_c2m8k5": (2, 8, 5, 2, 94, 194, 0, 128),
    "small_c4m4k1": (4, 4, 1, 4, 33, 133, 0, 64),
    "small_c4to2": (4, 4, 3, 2, 34, 134, 0, 64),
    "small_dup_c2m4k3": (2, 4, 3, 2, 35, 135, 0, 64),
}
CFG5 = dict(c=16, m=32, kappa=3, seed_img=1003, seed_filts=(2003, 2004, 2005), weight_kind=1, s=16384)
# multi-shard image mode (conv_image_shards conv.cpp:261-264): t = c m^2 / s input
# shards, n_out = c_out m^2 / s output shards
MS_CASES = {
    "ms_cfg1_c8": (8, 32, 3, 8, 1010, 2010, 0, 4096),       # t = 2, n_out = 2
    "ms_cfg1_c8to4": (8, 32, 3, 4, 1011, 2011, 0, 4096),    # t = 2, n_out = 1
    "ms_cfg1_c4to8": (4, 32, 3, 8, 1012, 2012, 0, 4096),    # t = 1, n_out = 2
    "ms_cfg3_c32": (32, 32, 3, 32, 1013, 2013, 0, 16384),   # t = 2, n_out = 2
}
# 2x2 average pooling (pool.cpp:291-297): (c, m, s, seed), image mode without duplication
POOL_CASES = {
    "pool_cfg1_c4m32": (4, 32, 4096, 1040),    # t = 1: duplicated x4 after pooling
    "pool_cfg1_c8m32": (8, 32, 4096, 1041),    # t = 2
    "pool_cfg1_c16m32": (16, 32, 4096, 1042),  # t = 4
    "pool_cfg3_c16m32": (16, 32, 16384, 1043), # cfg3 feature map, t = 1
}
# pool / subsample_stride2 over every packing (pool.cpp:238-306): (c, m, s, window, output_scale, seed)
DS_CASES = {
    "ds_cfg1_c2m128_pool": (2, 128, 4096, 1, 1.0, 1050),   # channel shards (pc 4, 32 rows) -> 2 image shards
    "ds_cfg1_c1m256_pool": (1, 256, 4096, 1, 1.0, 1051),   # channel shards (pc 16) -> channel shards (pc 4)
    "ds_cfg1_c1m128_pool": (1, 128, 4096, 1, 1.0, 1052),   # channel shards -> one full image shard
    "ds_cfg2_c1m128_pool": (1, 128, 8192, 1, 1.0, 1053),   # channel shards -> image shard duplicated x2
    "ds_cfg1_c2m32_pool": (2, 32, 4096, 1, 1.0, 1054),     # duplicated input (d 2) -> rep 4, d 8
    "ds_cfg1_c8m32_pool_sc": (8, 32, 4096, 1, 0.5, 1055),  # output_scale on the vertical masks
    "ds_cfg1_c4m32_s2": (4, 32, 4096, 0, 1.0, 1056),       # stride-2, one shard
    "ds_cfg1_c16m32_s2": (16, 32, 4096, 0, 1.0, 1057),     # stride-2, four shards
    "ds_cfg1_c2m128_s2": (2, 128, 4096, 0, 1.0, 1058),     # stride-2, channel -> image shards
    "ds_cfg1_c1m256_s2": (1, 256, 4096, 0, 1.0, 1059),     # stride-2, channel -> channel shards
}
# linear head: (c, m, s, out_features, seed)
LIN_CASES = {
    "lin_cfg1_c4m32": (4, 32, 4096, 4, 1030),     # one shard
    "lin_cfg1_c8m32": (8, 32, 4096, 3, 1031),     # two image shards
    "lin_cfg1_c2m16": (2, 16, 4096, 3, 1032),     # duplicated single shard (d = 8)
    "lin_cfg1_c1m128": (1, 128, 4096, 2, 1033),   # four channel shards
}
# channel-shard mode (conv_channel_shards conv.cpp:273-362): m^2 > s, pc = m^2 / s shards per channel
CS_CASES = {
    "cs_cfg1_c2m128": (2, 128, 3, 2, 1020, 2020, 0, 4096),     # pc = 4
    "cs_cfg1_c2to4m128": (2, 128, 3, 4, 1021, 2021, 0, 4096),  # pc = 4, 16 output shards
    "cs_cfg3_c1m256k5": (1, 256, 5, 2, 1022, 2022, 0, 16384),  # pc = 4, 5x5
}


# Chebyshev activation (act.cpp:151-162): (func, degree, bound, prescaled, level, slots, seed); the
# input is uniform on [-bound, bound] (divided by bound when prescaled), slots = the config's slots
CHEB_CASES = {
    "cheb_cfg3_gelu27_pre": ("gelu", 27, 10.0, 1, 12, 16384, 1050),  # test_act.cpp:78-96
    "cheb_cfg3_gelu59_raw": ("gelu", 59, 16.0, 0, 12, 16384, 1051),  # the degree-59 table entry
    "cheb_cfg3_relu27_raw": ("relu", 27, 16.0, 0, 12, 16384, 1052),
    "cheb_cfg3_relu16_raw": ("relu", 16, 4.0, 0, 7, 16384, 1053),    # exact power of two: the p == d peel
    "cheb_cfg1_gelu7_raw": ("gelu", 7, 4.0, 0, 4, 4096, 1054),      # cfg1: ends at level 0
    "cheb_cfg1_identity": ("ident", 1, 4.0, 0, 4, 4096, 1055),     # test_act.cpp:99-110
    "cheb_cfg1_const": ("const", 0, 4.0, 0, 4, 4096, 1056),        # degree 0
}
CHEB_KEEP = 2048  # stored output slots per case


def cheb_func(name):
    if name == "gelu":
        return lambda x: x * 0.5 * (1.0 + math.erf(x / math.sqrt(2.0)))  # oracle.cpp:78-81
    if name == "relu":
        return lambda x: x if x > 0.0 else 0.0
    return lambda x: x


def cheb_case(name):
    func, deg, bound, pre, level, s, seed = CHEB_CASES[name]
    x = np.random.default_rng(seed).uniform(-bound, bound, s)
    if pre:
        x = x / bound
    if func == "ident":
        co = np.array([0.0, bound])
    elif func == "const":
        co = np.array([0.7])
    else:
        co = po.ref_cheb_interpolate(cheb_func(func), deg, bound)
    return x, co


def main():
    R = po.ref()
    out = {}
    for name, (c, m, k, co, si, sf, wk, s) in CONV_CASES.items():
        img, filt = po.make_inputs(c, m, k, co, si, sf, wk, use_ref=True)
        res = {}
        for plan in (0, 1, 2):
            res[plan] = po.ref_conv(c, m, k, co, img, filt, plan, s)
        assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[1][0], res[2][0])
        oracle = np.zeros(co * m * m)
        R.ref_oracle_conv(c, m, k, co, img.ctypes.data_as(po.dp), filt.ctypes.data_as(po.dp), 1,
                          oracle.ctypes.data_as(po.dp))
        out[f"{name}/params"] = np.array([c, m, k, co, si, sf, wk, s], dtype=np.int64)
        out[f"{name}/img"] = img if img.size <= 4096 else img[:64]
        out[f"{name}/img_sum"] = np.array([img.sum(), np.abs(img).sum()])
        out[f"{name}/filt"] = filt
        out[f"{name}/slots"] = res[2][0]
        if not np.array_equal(res[2][1], res[2][0][: co * m * m]):
            out[f"{name}/image"] = res[2][1]
        # textbook oracle agrees to ~1e-14 (summation order differs); keep its max deviation
        out[f"{name}/oracle_dev"] = np.array([np.abs(oracle - res[2][1]).max()])
        if oracle.size <= 4096:
            out[f"{name}/oracle_conv"] = oracle
        for plan in (0, 1, 2):
            out[f"{name}/ledger{plan}"] = res[plan][2]
        out[f"{name}/level_drop"] = np.array([res[2][3]])
    for name, (c, m, k, co, si, sf, wk, s) in MS_CASES.items():
        img, filt = po.make_inputs(c, m, k, co, si, sf, wk, use_ref=True)
        slots, image, ledger, drop = po.ref_conv_shards(c, m, k, co, img, filt, s)
        out[f"{name}/params"] = np.array([c, m, k, co, si, sf, wk, s], dtype=np.int64)
        out[f"{name}/img_sum"] = np.array([img.sum(), np.abs(img).sum()])
        out[f"{name}/slots"] = slots
        out[f"{name}/ledger"] = ledger
    for name, (c, m, k, co, si, sf, wk, s) in CS_CASES.items():
        img, filt = po.make_inputs(c, m, k, co, si, sf, wk, use_ref=True)
        slots, image, ledger, drop = po.ref_conv_channel(c, m, k, co, img, filt, s)
        out[f"{name}/params"] = np.array([c, m, k, co, si, sf, wk, s], dtype=np.int64)
        out[f"{name}/img_sum"] = np.array([img.sum(), np.abs(img).sum()])
        out[f"{name}/slots"] = slots
        out[f"{name}/ledger"] = ledger
    # the linear head (dense.cpp:34-75) and slot_sum (dense.cpp:23-30)
    for name, (c, m, s, no, si) in LIN_CASES.items():
        img, _ = po.make_inputs(c, m, 1, 1, si, 0, 0, use_ref=True)
        rng = np.random.default_rng(si)
        w = rng.uniform(-1, 1, no * c * m * m)
        b = rng.uniform(-1, 1, no)
        slots, ledger, t = po.ref_linear(c, m, img, w, b, s)
        out[f"{name}/params"] = np.array([c, m, s, no, si, t], dtype=np.int64)
        out[f"{name}/w_sum"] = np.array([w.sum()])
        out[f"{name}/slots"] = slots[:no]
        out[f"{name}/ledger"] = ledger
    for name, (c, m, s, si) in POOL_CASES.items():
        img, _ = po.make_inputs(c, m, 1, 1, si, 0, 0, use_ref=True)
        slots, meta, tau, ledger = po.ref_pool(c, m, img, s)
        out[f"{name}/params"] = np.array([c, m, s, si], dtype=np.int64)
        out[f"{name}/slots"] = slots
        out[f"{name}/meta"] = meta
        out[f"{name}/tau"] = tau
        out[f"{name}/ledger"] = ledger
    for name, (c, m, s, window, osc, si) in DS_CASES.items():
        img, _ = po.make_inputs(c, m, 1, 1, si, 0, 0, use_ref=True)
        slots, meta, tau, ledger = po.ref_downsample(c, m, img, s, window, osc)
        out[f"{name}/params"] = np.array([c, m, s, window, osc, si], dtype=np.float64)
        out[f"{name}/slots"] = slots
        out[f"{name}/meta"] = meta
        out[f"{name}/tau"] = tau
        out[f"{name}/ledger"] = ledger
    for name, (func, deg, bound, pre, level, s, seed) in CHEB_CASES.items():
        x, co = cheb_case(name)
        y, lv, depth, ledger = po.ref_eval_chebyshev(x, level, co, bound, pre)
        out[f"{name}/params"] = np.array([deg, bound, pre, level, s, seed], dtype=np.float64)
        out[f"{name}/x_sum"] = np.array([x.sum(), np.abs(x).sum()])
        out[f"{name}/coeffs"] = co
        out[f"{name}/slots"] = y[:CHEB_KEEP]
        out[f"{name}/meta"] = np.array([lv, depth], dtype=np.int64)
        out[f"{name}/ledger"] = ledger
    try:
        po.ref_eval_chebyshev(np.full(16, 0.1), 3, po.ref_cheb_interpolate(cheb_func("gelu"), 27, 10.0), 10.0, 1)
        raise AssertionError("expected the level check to throw")
    except RuntimeError as e:
        out["cheb_level_error"] = np.frombuffer(str(e).encode(), dtype=np.uint8)
    rng = np.random.default_rng(77)
    vec = rng.uniform(-1, 1, 4096)
    out["slot_sum/vec_sum"] = np.array([vec.sum()])
    for block in (1, 4, 64, 4096):
        out[f"slot_sum/block{block}"] = po.ref_slot_sum(vec, block)
    # cfg5: three stacked layers, each input = previous output image
    x, _ = po.make_inputs(CFG5["c"], CFG5["m"], CFG5["kappa"], CFG5["c"], CFG5["seed_img"], 0, 0, use_ref=True)
    out["cfg5/img_sum"] = np.array([x.sum(), np.abs(x).sum()])
    for li, sf in enumerate(CFG5["seed_filts"]):
        _, filt = po.make_inputs(CFG5["c"], CFG5["m"], CFG5["kappa"], CFG5["c"], 0, sf, CFG5["weight_kind"],
                                 use_ref=True)
        slots, image, ledger, drop = po.ref_conv(CFG5["c"], CFG5["m"], CFG5["kappa"], CFG5["c"], x, filt, 2,
                                                 CFG5["s"])
        out[f"cfg5/filt{li}"] = filt
        out[f"cfg5/out{li}"] = slots
        x = image
    # rotation decompositions (rot.cpp:21-94)
    import ctypes as C
    for s in (4096, 8192):
        lens = np.zeros((2, s), dtype=np.int8)
        sums = np.zeros((2, s), dtype=np.int32)
        first = np.zeros((2, 1024, 16), dtype=np.int16)
        buf = (C.c_long * 64)()
        for strat in (0, 1):
            for n in range(s):
                k = R.ref_decompose(strat, n, s, buf, 64)
                lens[strat, n] = k
                sums[strat, n] = sum(buf[i] for i in range(k))
                if n < 1024:
                    first[strat, n, :k] = [buf[i] for i in range(k)]
        out[f"decomp{s}/lens"] = lens
        out[f"decomp{s}/sums"] = sums
        out[f"decomp{s}/steps_lt1024"] = first
    ml = np.zeros(4096, dtype=np.uint64)
    R.ref_min_lengths(4095, 4096, ml.ctypes.data_as(po.u64p))
    out["minlen4096"] = ml.astype(np.int8)
    # planner (rot.cpp:96-129): cfg2 amounts 1..127 and the 3x3 stencil (m = 32)
    def plan(amounts, same, s, strat):
        n = len(amounts)
        a = (C.c_long * n)(*amounts)
        ss = (C.c_int * n)(*same)
        steps = (C.c_long * (64 * n))()
        ns = (C.c_int * n)()
        g = (C.c_int * n)()
        gh = (C.c_int * n)()
        tot = R.ref_plan_rotations(a, ss, n, s, strat, steps, ns, g, gh)
        return tot, np.array(list(ns)), np.array(list(g)), np.array(list(gh))
    amounts = list(range(1, 128))
    stencil = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1)]
    for strat in (0, 1, 2):
        tot, ns, g, gh = plan(amounts, [0] * 127, 8192, strat)
        out[f"plan_cfg2/strat{strat}/total"] = np.array([tot])
        out[f"plan_cfg2/strat{strat}/nsteps"] = ns
        tot, ns, g, gh = plan(stencil, [0] + [1] * 8, 8192, strat)
        out[f"plan_stencil/strat{strat}/total"] = np.array([tot])
        out[f"plan_stencil/strat{strat}/nsteps"] = ns
        out[f"plan_stencil/strat{strat}/groups"] = g
        out[f"plan_stencil/strat{strat}/hoisted"] = gh
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
