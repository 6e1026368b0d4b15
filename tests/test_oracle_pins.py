"""Pins the oracle's C restatement (oracle/emu_ref.c, mt19937.c) against the
reference's own outputs: the committed golden fixtures (generated from the
compiled, unmodified reference by tests/golden/make_golden.py) and, where
oracle/_ref was built, the live reference library."""
import numpy as np
import pytest

CASES = ["cfg1", "cfg3", "cfg4", "small_c4m4k3", "small_c2m8k5", "small_c4m4k1", "small_c4to2",
         "small_dup_c2m4k3"]


def params(golden, name):
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    return c, m, k, co, si, sf, wk, s


@pytest.mark.parametrize("name", CASES)
def test_inputs_regenerate_bit_exact(oracle, golden, name):
    c, m, k, co, si, sf, wk, s = params(golden, name)
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    ref_img = golden[f"{name}/img"]
    assert np.array_equal(img[: ref_img.size], ref_img)
    assert np.array_equal(np.array([img.sum(), np.abs(img).sum()]), golden[f"{name}/img_sum"])
    assert np.array_equal(filt, golden[f"{name}/filt"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("plan", [0, 1, 2])
def test_emulator_conv_bit_exact_vs_reference(oracle, golden, name, plan):
    """conv_plan / convolve slots (reference conv.cpp:109-211) reproduced bit for bit."""
    c, m, k, co, si, sf, wk, s = params(golden, name)
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    if s > c * m * m:  # pack() duplicates the channel sequence (pack.cpp:19-33)
        img = np.tile(img, s // (c * m * m))
    out = oracle.emu_conv_slots(c, m, k, co, s, img[: c * m * m], filt, plan)
    assert np.array_equal(out, golden[f"{name}/slots"])


@pytest.mark.parametrize("name", ["small_c4m4k3", "small_c2m8k5", "small_c4m4k1", "small_c4to2", "cfg1"])
def test_textbook_conv_matches_reference_oracle(oracle, golden, name):
    c, m, k, co, si, sf, wk, s = params(golden, name)
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    out = oracle.emu_oracle_conv(c, m, k, co, img, filt)
    assert np.array_equal(out, golden[f"{name}/oracle_conv"])
    # and the slot schedule agrees with the textbook conv (reference test_conv.cpp:86)
    image = golden.get(f"{name}/image", golden[f"{name}/slots"][: co * m * m])
    assert np.abs(image - out).max() < 1e-12


def test_cfg5_stack_bit_exact(oracle, golden):
    x, _ = oracle.make_inputs(16, 32, 3, 16, 1003, 0, 0)
    assert np.array_equal(np.array([x.sum(), np.abs(x).sum()]), golden["cfg5/img_sum"])
    for li, sf in enumerate((2003, 2004, 2005)):
        _, filt = oracle.make_inputs(16, 32, 3, 16, 0, sf, 1)
        assert np.array_equal(filt, golden[f"cfg5/filt{li}"])
        x = oracle.emu_conv_slots(16, 32, 3, 16, 16384, x, filt, 2)
        assert np.array_equal(x, golden[f"cfg5/out{li}"])


def test_rotation_kats(oracle):
    """reference test_emu.cpp:13-26"""
    v = np.array([1.0, 2, 3, 4])
    out = np.zeros(4)
    for k, want in [(1, [2, 3, 4, 1]), (-1, [4, 1, 2, 3]), (5, [2, 3, 4, 1]), (0, [1, 2, 3, 4])]:
        oracle.lib().emu_rotate(v.ctypes.data_as(oracle.dp), out.ctypes.data_as(oracle.dp), 4, k)
        assert out.tolist() == want


def test_single_channel_kats(oracle):
    """reference test_conv.cpp:60-79 (identity, x2 scale, all-ones -> {10,10,10,10})"""
    ch = np.array([1.0, 2, 3, 4])
    assert oracle.emu_conv_slots(1, 2, 1, 1, 4, ch, np.array([2.0]), 0).tolist() == [2, 4, 6, 8]
    ident = np.zeros(9)
    ident[4] = 1.0
    assert oracle.emu_conv_slots(1, 2, 3, 1, 4, ch, ident, 0).tolist() == [1, 2, 3, 4]
    assert oracle.emu_conv_slots(1, 2, 3, 1, 4, ch, np.ones(9), 0).tolist() == [10, 10, 10, 10]


@pytest.mark.parametrize("s", [4096, 8192])
def test_decompositions_vs_reference(oracle, golden, s):
    lens, sums, first = golden[f"decomp{s}/lens"], golden[f"decomp{s}/sums"], golden[f"decomp{s}/steps_lt1024"]
    for strat in (0, 1):
        for n in range(s):
            st = oracle.emu_decompose(strat, n, s)
            assert len(st) == lens[strat, n] and sum(st) == sums[strat, n]
            if n < 1024:
                assert st == [int(x) for x in first[strat, n, : len(st)]]


def test_decomposition_kats(oracle):
    """reference test_rot.cpp:12-29"""
    assert oracle.emu_decompose(0, 127, 4096) == [64, 32, 16, 8, 4, 2, 1]
    assert oracle.emu_decompose(1, 127, 4096) == [128, -1]
    assert oracle.emu_decompose(1, 96, 4096) == [64, 32]
    assert oracle.emu_decompose(1, 5, 4096) == [4, 1]
    assert oracle.emu_decompose(1, 0, 4096) == []


def test_min_lengths_vs_reference(oracle, golden):
    ml = oracle.emu_min_lengths(4095, 4096)
    assert np.array_equal(ml.astype(np.int8), golden["minlen4096"])
    # greedy signed is BFS-minimal for every n < 4096 (acceptance.cpp:245-259)
    for n in range(4096):
        assert len(oracle.emu_decompose(1, n, 4096)) == ml[n]


def test_planner_counts_vs_reference(golden):
    # survey-reported values of the reference planner
    assert int(golden["plan_cfg2/strat0/total"][0]) == 448
    assert int(golden["plan_cfg2/strat1/total"][0]) == 355
    assert [int(golden[f"plan_stencil/strat{s}/total"][0]) for s in (0, 1, 2)] == [51, 16, 8]


def test_live_reference_if_built(oracle, golden):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here (no /root/reference)")
    c, m, k, co, si, sf, wk, s = params(golden, "cfg1")
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk, use_ref=True)
    slots, _, ledger, drop = oracle.ref_conv(c, m, k, co, img, filt, 2, s)
    assert np.array_equal(slots, golden["cfg1/slots"])
    assert np.array_equal(ledger, golden["cfg1/ledger2"]) and drop == 1


@pytest.mark.parametrize("name", ["ms_cfg1_c8", "ms_cfg1_c8to4", "ms_cfg1_c4to8", "ms_cfg3_c32"])
def test_multishard_restatement_bit_exact(oracle, golden, name):
    """emu_conv_shards_slots (conv_image_mode with t input shards / n_out output shards,
    SURVEY §8(f) 1) == the reference's conv_image_shards slots, bit for bit."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    assert np.isclose(img.sum(), golden[f"{name}/img_sum"][0])
    got = oracle.emu_conv_shards_slots(c, m, k, co, s, img, filt)
    assert np.array_equal(got, golden[f"{name}/slots"])
    # and it is the textbook same-padding conv of the image
    want = oracle.emu_oracle_conv(c, m, k, co, img, filt)
    assert np.abs(got.ravel()[: co * m * m] - want).max() < 1e-12


@pytest.mark.parametrize("name", ["cs_cfg1_c2m128", "cs_cfg1_c2to4m128", "cs_cfg3_c1m256k5"])
def test_channel_shard_restatement_bit_exact(oracle, golden, name):
    """emu_conv_channel_slots (channel-shard mode, m^2 > slots, in-shard + neighbour-spill masks)
    == the reference's conv_channel_shards slots, bit for bit."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    assert np.isclose(img.sum(), golden[f"{name}/img_sum"][0])
    got = oracle.emu_conv_channel_slots(c, m, k, co, s, img, filt)
    assert np.array_equal(got, golden[f"{name}/slots"])
    want = oracle.emu_oracle_conv(c, m, k, co, img, filt)
    assert np.abs(got.ravel() - want).max() < 1e-12


def test_slot_sum_restatement_bit_exact(golden):
    """rotate-and-add block sums (reference slot_sum, dense.cpp:23-30) restated with numpy,
    bit-exact against the reference for block 1, 4, 64 and the whole vector."""
    vec = np.random.default_rng(77).uniform(-1, 1, 4096)
    assert vec.sum() == golden["slot_sum/vec_sum"][0]
    for block in (1, 4, 64, 4096):
        acc = vec.copy()
        step = 1
        while step < block:
            acc = acc + np.roll(acc, -step)
            step *= 2
        assert np.array_equal(acc, golden[f"slot_sum/block{block}"])


@pytest.mark.parametrize("name", ["lin_cfg1_c4m32", "lin_cfg1_c8m32", "lin_cfg1_c2m16", "lin_cfg1_c1m128"])
def test_linear_reference_is_wx_plus_b(oracle, golden, name):
    """the reference's linear() over every packing (one shard, image shards, duplicated shard,
    channel shards) equals W x + b; rotations = out x shards x log2(s) (test_dense.cpp:137-148)."""
    c, m, s, no, si, t = (int(x) for x in golden[f"{name}/params"])
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    rng = np.random.default_rng(si)
    w = rng.uniform(-1, 1, no * c * m * m)
    b = rng.uniform(-1, 1, no)
    assert np.isclose(w.sum(), golden[f"{name}/w_sum"][0])
    want = w.reshape(no, -1) @ img + b
    assert np.abs(golden[f"{name}/slots"] - want).max() < 1e-12
    assert int(golden[f"{name}/ledger"][0]) == no * t * int(np.log2(s))


def _pool_restatement(img, c, m, s):
    """numpy restatement of the reference's pool() on an image-mode map (pool.cpp:10-104,
    167-226, 280-289) through the rotation-of-mask form used by the GPU path."""
    block, bn = m * m, (m // 2) ** 2
    t = c * block // s
    rot = lambda v, k: np.roll(v, -k)
    shards = [img[u * s:(u + 1) * s] for u in range(t)]

    def wmask(kk, ll):
        v = np.zeros(s)
        for b in range(s // block):
            for i in range(m - kk):
                v[b * block + i * m: b * block + i * m + (m - ll)] = 0.25
        return v
    W = [sum(wmask(kk, ll) * rot(x, kk * m + ll) for kk, ll in ((0, 0), (0, 1), (1, 0), (1, 1))) for x in shards]
    H, V = [], []
    for x in W:
        acc = 0
        for i in range(m // 2):
            mk = np.zeros(s)
            mk[2 * i::m] = 1.0
            acc = acc + rot(mk, i) * rot(x, i)
        H.append(acc)
    for x in H:
        acc = 0
        for j in range(m // 2):
            mv = np.zeros(s)
            for b in range(s // block):
                mv[b * block + 2 * j * m: b * block + 2 * j * m + m // 2] = 1.0
            acc = acc + rot(mv, 3 * j * m // 2) * rot(x, 3 * j * m // 2)
        V.append(acc)
    if t == 1:
        base = V[0]
        return [base + sum(rot(base, -e * bn) for e in range(1, 4))]
    if t == 2:
        sm = V[0] + rot(V[1], -2 * bn)
        return [sm + rot(sm, -bn)]
    return [V[4 * w] + sum(rot(V[4 * w + q], -q * bn) for q in range(1, 4)) for w in range(t // 4)]


@pytest.mark.parametrize("name", ["pool_cfg1_c4m32", "pool_cfg1_c8m32", "pool_cfg1_c16m32", "pool_cfg3_c16m32"])
def test_pool_restatement_matches_reference(oracle, golden, name):
    """the rotation-of-mask form of pooling (what the GPU runs) reproduces the reference's
    pool() shards to 1e-12 (summation order differs), and the reference pools correctly."""
    c, m, s, si = (int(x) for x in golden[f"{name}/params"])
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    got = _pool_restatement(img, c, m, s)
    want = golden[f"{name}/slots"]
    assert len(got) == want.shape[0]
    for a, b in zip(got, want):
        assert np.abs(a - b).max() < 1e-12
    # logical check: pooled channel tau[g] at physical block g of the first shard
    meta, tau = golden[f"{name}/meta"], golden[f"{name}/tau"]
    mn = m // 2
    x = img.reshape(c, m, m)
    pooled = 0.25 * (x[:, 0::2, 0::2] + x[:, 1::2, 0::2] + x[:, 0::2, 1::2] + x[:, 1::2, 1::2])
    rep = int(meta[3])
    for g in range(min(c * rep, s // (mn * mn))):
        if g % rep:
            continue
        ch = int(tau[(g // rep) % c])
        assert np.abs(want[0][g * mn * mn:(g + 1) * mn * mn] - pooled[ch].ravel()).max() < 1e-12


DS = ["ds_cfg1_c2m128_pool", "ds_cfg1_c1m256_pool", "ds_cfg1_c1m128_pool", "ds_cfg2_c1m128_pool",
      "ds_cfg1_c2m32_pool", "ds_cfg1_c8m32_pool_sc", "ds_cfg1_c4m32_s2", "ds_cfg1_c16m32_s2",
      "ds_cfg1_c2m128_s2", "ds_cfg1_c1m256_s2"]


def packed(img, c, m, s):
    """pack(img, s) slot vectors (pack.cpp:7-49): image mode duplicates a small image d times."""
    block = m * m
    d = s // (block * c) if block <= s and block * c < s else 1
    flat = np.tile(img, d)
    return list(flat.reshape(-1, s)), d


@pytest.mark.parametrize("name", DS)
def test_downsample_restatement_matches_reference(oracle, golden, name):
    """pool() / subsample_stride2() over channel shards, duplicated inputs and output scales:
    the rotation-of-mask restatement (what the GPU runs) reproduces the reference's shards
    (1e-12) and packing metadata, and the result is the average-pooled / subsampled image."""
    c, m, s, window, osc, si = golden[f"{name}/params"]
    c, m, s, window, si = int(c), int(m), int(s), int(window), int(si)
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    xs, d_in = packed(img, c, m, s)
    got, tau, rep, d, mode = oracle.downsample_restated(oracle.NumpyOps, xs, c, m, s, bool(window), float(osc),
                                                        d_in=d_in)
    want, meta = golden[f"{name}/slots"], golden[f"{name}/meta"]
    assert len(got) == want.shape[0] == int(meta[5])
    assert (rep, d, mode) == (int(meta[3]), int(meta[2]), int(meta[4]))
    assert np.array_equal(tau, golden[f"{name}/tau"].astype(np.int64))
    for a, b in zip(got, want):
        assert np.abs(a - b).max() < 1e-12
    # logical check on the reference's output: unpack and compare with the numpy pooled image
    x = img.reshape(c, m, m)
    if window:
        want_img = 0.25 * (x[:, 0::2, 0::2] + x[:, 1::2, 0::2] + x[:, 0::2, 1::2] + x[:, 1::2, 1::2])
    else:
        want_img = x[:, 0::2, 0::2].copy()
    want_img *= float(osc)
    mn = m // 2
    if mode == 1:  # channel shards: channel-major, rows_per_shard rows each
        flat = np.concatenate(list(want))
        assert np.abs(flat[: c * mn * mn] - want_img.ravel()).max() < 1e-12
    else:
        bn = mn * mn
        for ph in range(min(c * rep, s // bn) if len(want) == 1 else c):
            if ph % rep:
                continue
            sh, pos = divmod(ph // rep, s // bn) if len(want) > 1 else (0, ph)
            ch = int(tau[ph // rep])
            assert np.abs(want[sh][pos * bn:(pos + 1) * bn] - want_img[ch].ravel()).max() < 1e-12


def test_downsample_steps_cover_restatement():
    """downsample_steps lists every rotation the restatement performs (the Galois key set)."""
    for c, m, s, w in [(2, 128, 4096, 1), (1, 256, 4096, 0), (4, 32, 4096, 1), (1, 128, 8192, 1)]:
        used = set()

        class Rec(oracle_mod().NumpyOps):
            @staticmethod
            def lintrans(srcs, terms):
                used.update(a % s for _, a, _ in terms if a % s)
                return oracle_mod().NumpyOps.lintrans(srcs, terms)

            @staticmethod
            def rotate(x, k):
                if k % s:
                    used.add(k % s)
                return np.roll(x, -k)
        img = np.random.default_rng(0).uniform(-1, 1, c * m * m)
        xs, d_in = packed(img, c, m, s)
        oracle_mod().downsample_restated(Rec, xs, c, m, s, bool(w), d_in=d_in)
        assert used <= set(oracle_mod().downsample_steps(c, m, s, bool(w)))


def oracle_mod():
    import pyoracle
    return pyoracle


CHEB = ["cheb_cfg3_gelu27_pre", "cheb_cfg3_gelu59_raw", "cheb_cfg3_relu27_raw", "cheb_cfg3_relu16_raw",
        "cheb_cfg1_gelu7_raw", "cheb_cfg1_identity", "cheb_cfg1_const"]


def cheb_input(golden, name):
    """the case's input slots (seeded uniform on [-B, B], / B when prescaled), checked against the fixture"""
    deg, bound, pre, level, s, seed = golden[f"{name}/params"]
    x = np.random.default_rng(int(seed)).uniform(-bound, bound, int(s))
    if pre:
        x = x / bound
    assert np.array_equal(np.array([x.sum(), np.abs(x).sum()]), golden[f"{name}/x_sum"])
    return x, int(deg), float(bound), bool(pre), int(level)


@pytest.mark.parametrize("name", [n for n in CHEB if "gelu" in n or "relu" in n])
def test_cheb_interpolate_restatement_bit_exact(oracle, golden, name):
    """pyoracle.cheb_interpolate (restating act.cpp:90-113) = the reference's coefficients bit for bit."""
    import math
    deg, bound = int(golden[f"{name}/params"][0]), float(golden[f"{name}/params"][1])
    if "gelu" in name:
        f = lambda x: x * 0.5 * (1.0 + math.erf(x / math.sqrt(2.0)))  # noqa: E731
    else:
        f = lambda x: x if x > 0.0 else 0.0  # noqa: E731
    assert np.array_equal(oracle.cheb_interpolate(f, deg, bound), golden[f"{name}/coeffs"])


@pytest.mark.parametrize("name", CHEB)
def test_cheb_series_equals_clenshaw(oracle, golden, name):
    """The reference's power-of-two split evaluation (act.cpp:49-82) equals the plain Clenshaw
    evaluation slotwise (test_act.cpp:78-96), and its level bookkeeping is bits(d) (+1 raw)."""
    x, deg, bound, pre, level = cheb_input(golden, name)
    want = golden[f"{name}/slots"]
    co = golden[f"{name}/coeffs"]
    xr = x[: want.size] * (bound if pre else 1.0)
    assert np.abs(oracle.cheb_eval(co, bound, xr) - want).max() < 1e-9
    lv, depth = golden[f"{name}/meta"]
    assert lv == (level - (int(deg).bit_length() + (0 if pre else 1)) if deg > 0 else level)


def test_cheb_level_error_text(golden):
    assert bytes(golden["cheb_level_error"]).decode() == "insufficient level for activation: bootstrap required"


def test_cheb_ckks_composition_matches_reference(oracle, golden):
    """The golden model's ciphertext composition (relinearised products, scale targeting)
    decrypts to the reference's eval_chebyshev slots (cfg1: degree 7, unprescaled)."""
    name = "cheb_cfg1_gelu7_raw"
    x, deg, bound, pre, level = cheb_input(golden, name)
    ck = oracle.CKKS(13, [60] + [40] * 4, [60], 40)
    ck.keygen(7)
    ct = ck.encrypt(ck.encode(x, ck.scale, level), level, 9000)
    out, lv, sc = ck.eval_chebyshev(ct, level, ck.scale, golden[f"{name}/coeffs"], bound, pre)
    assert lv == golden[f"{name}/meta"][0] and sc == ck.scale
    want = golden[f"{name}/slots"]
    assert np.abs(ck.decrypt(out, lv, sc)[: want.size] - want).max() < 1e-6
