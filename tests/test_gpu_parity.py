"""GPU parity: every op of libfheconv (through the C ABI) is bit-exact with
the CPU golden model (oracle/ckks_ref.c) on the same seeds, and decrypted
conv outputs agree with the reference's conv_plan slots within 1e-6
(BASELINE north star). Tolerance 1e-6 absolute on decrypted slots."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-6
KEY_SEED, ENC_SEED = 7, 9000


class Pair:
    """GPU context + CPU golden model with the same parameters and keys."""

    def __init__(self, oracle, name):
        from paper_2306_09189_b200 import CONFIGS, Context
        p = CONFIGS[name]
        self.ctx = Context.from_config(name)
        self.ck = oracle.CKKS(p["log_n"], p["q_bits"], p["p_bits"], p["log_scale"])
        self.ctx.keygen(KEY_SEED)
        self.ck.keygen(KEY_SEED)
        self.top = self.ctx.max_level


_pairs = {}


def pair(oracle, name):
    if name not in _pairs:
        _pairs[name] = Pair(oracle, name)
    return _pairs[name]


@pytest.fixture(scope="module")
def p1(oracle):
    return pair(oracle, "cfg1")


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def test_primes_match_golden_model(oracle):
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        p = pair(oracle, name)
        assert p.ctx.primes == p.ck.primes


def test_encode_encrypt_bit_exact(p1):
    z = rnd(p1.ctx.slots, 1)
    pt = p1.ctx.encode(z)
    ptr = p1.ck.encode(z, p1.ck.scale, p1.top)
    assert np.array_equal(pt.residues(), ptr)
    ptp = p1.ctx.encode(z, with_special=True)
    assert np.array_equal(ptp.residues(), p1.ck.encode(z, p1.ck.scale, p1.top, with_p=True))
    ct = p1.ctx.encrypt(pt, ENC_SEED)
    assert np.array_equal(ct.residues(), p1.ck.encrypt(ptr, p1.top, ENC_SEED))
    assert np.abs(p1.ctx.decrypt(ct) - z).max() < 1e-8
    # lower level + short slot vector (Engine::encode accepts any power of two)
    pt2 = p1.ctx.encode(z[:256], level=2)
    assert np.array_equal(pt2.residues(), p1.ck.encode(z[:256], p1.ck.scale, 2))


def test_galois_keys_bit_exact(p1):
    p1.ctx.gen_galois_keys([1, 33, -1])
    for k in (1, 33, -1):
        assert np.array_equal(p1.ctx.galois_key(k), p1.ck.galois_key(p1.ck.galois(k)))


@pytest.mark.parametrize("k", [1, -1, 33, 4095, -4096, 0, 8192])
def test_rotate_bit_exact(p1, k):
    p1.ctx.gen_galois_keys([k])
    z = rnd(p1.ctx.slots, 2)
    ct = p1.ctx.encrypt(p1.ctx.encode(z), ENC_SEED)
    ctr = p1.ck.encrypt(p1.ck.encode(z, p1.ck.scale, p1.top), p1.top, ENC_SEED)
    r = p1.ctx.rotate(ct, k)
    assert np.array_equal(r.residues(), p1.ck.rotate(ctr, p1.top, k))
    assert np.abs(p1.ctx.decrypt(r) - np.roll(z, -k)).max() < TOL


def test_rotate_hoisted_bit_exact(p1):
    ks = [1, -1, 32, -32, 33, -33, 31, -31, 0]
    p1.ctx.gen_galois_keys(ks)
    z = rnd(p1.ctx.slots, 3)
    ct = p1.ctx.encrypt(p1.ctx.encode(z), ENC_SEED)
    ctr = p1.ck.encrypt(p1.ck.encode(z, p1.ck.scale, p1.top), p1.top, ENC_SEED)
    outs = p1.ctx.rotate_hoisted(ct, ks)
    ref = p1.ck.rotate_hoisted(ctr, p1.top, ks)
    for i, k in enumerate(ks):
        assert np.array_equal(outs[i].residues(), ref[i])
        assert np.abs(p1.ctx.decrypt(outs[i]) - np.roll(z, -k)).max() < TOL


def test_elementwise_and_rescale_bit_exact(p1):
    a, b, w = rnd(p1.ctx.slots, 4), rnd(p1.ctx.slots, 5), rnd(p1.ctx.slots, 6)
    L = p1.top
    ca, cb = p1.ctx.encrypt(p1.ctx.encode(a), 11), p1.ctx.encrypt(p1.ctx.encode(b), 12)
    ra = p1.ck.encrypt(p1.ck.encode(a, p1.ck.scale, L), L, 11)
    rb = p1.ck.encrypt(p1.ck.encode(b, p1.ck.scale, L), L, 12)
    assert np.array_equal(p1.ctx.add(ca, cb).residues(), p1.ck.add(ra, rb, L))
    sub = p1.ctx.sub(ca, cb)
    assert np.abs(p1.ctx.decrypt(sub) - (a - b)).max() < 1e-8
    ql = float(p1.ctx.primes[L])
    pw, rw = p1.ctx.encode(w, scale=ql), p1.ck.encode(w, ql, L)
    m = p1.ctx.mul_plain(ca, pw)
    rm = p1.ck.mul_plain(ra, rw, L)
    assert np.array_equal(m.residues(), rm)
    rs = p1.ctx.rescale(m)
    assert rs.level == L - 1
    assert np.array_equal(rs.residues(), p1.ck.rescale(rm, L))
    assert np.abs(p1.ctx.decrypt(rs) - a * w).max() < 1e-7
    ap = p1.ctx.add_plain(ca, p1.ctx.encode(b))
    assert np.array_equal(ap.residues(), p1.ck.add_plain(ra, p1.ck.encode(b, p1.ck.scale, L), L))


def conv_case(oracle, golden, name):
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    return c, m, k, co, img, filt


@pytest.mark.parametrize("approach", [1, 2, 3, 4, 5])
def test_conv_cfg1_bit_exact_and_within_tolerance(oracle, golden, p1, approach):
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    layer = p1.ctx.conv_layer(c, co, m, k, filt)
    p1.ctx.gen_galois_keys(layer.steps())
    ct = p1.ctx.encrypt(p1.ctx.encode(img), ENC_SEED)
    ctr = p1.ck.encrypt(p1.ck.encode(img, p1.ck.scale, p1.top), p1.top, ENC_SEED)
    out = p1.ctx.conv2d(ct, layer, approach)
    ref, sc = p1.ck.conv(ctr, p1.top, c, m, k, co, filt, approach)
    assert out.level == p1.top - 1 and out.scale == sc
    assert np.array_equal(out.residues(), ref)
    err = np.abs(p1.ctx.decrypt(out) - golden["cfg1/slots"]).max()
    assert err < TOL, err


@pytest.mark.parametrize("approach", [1, 2, 3, 4, 5])
def test_conv_cfg3_bit_exact_and_within_tolerance(oracle, golden, approach):
    p = pair(oracle, "cfg3")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg3")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED)
    out = p.ctx.conv2d(ct, layer, approach)
    err = np.abs(p.ctx.decrypt(out) - golden["cfg3/slots"]).max()
    assert err < TOL, err
    ctr = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, ENC_SEED)
    assert np.array_equal(ct.residues(), ctr)
    ref, _ = p.ck.conv(ctr, p.top, c, m, k, co, filt, approach)
    assert np.array_equal(out.residues(), ref)


@pytest.mark.slow
@pytest.mark.parametrize("approach", [2, 4, 5])
def test_conv_cfg4_bit_exact_and_within_tolerance(oracle, golden, approach):
    p = pair(oracle, "cfg4")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg4")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED)
    out = p.ctx.conv2d(ct, layer, approach)
    err = np.abs(p.ctx.decrypt(out) - golden["cfg4/slots"]).max()
    assert err < TOL, err
    ctr = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, ENC_SEED)
    ref, _ = p.ck.conv(ctr, p.top, c, m, k, co, filt, approach)
    assert np.array_equal(out.residues(), ref)


def test_conv_auto_schedule_picks_fewer_decompositions(oracle, golden):
    p = pair(oracle, "cfg1")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED)
    a = p.ctx.conv2d(ct, layer, 0)
    b = p.ctx.conv2d(ct, layer, 5)  # c kappa = 12 fused baby steps, kappa = 3 giant steps
    assert np.array_equal(a.residues(), b.residues())


def test_conv_fused_schedule_runs_on_its_own_key_set(oracle, golden):
    """approach 5 needs exactly the rotations r m^2 + ll and kk m."""
    from paper_2306_09189_b200 import Context
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    ctx = Context.from_config("cfg1")
    ctx.keygen(7)
    layer = ctx.conv_layer(c, co, m, k, filt)
    steps = layer.steps(5)
    want = sorted(({r * m * m + ll for r in range(c) for ll in (-1, 0, 1)} | {-m, m}) - {0})
    assert sorted(steps) == want
    ctx.gen_galois_keys(steps)
    out = ctx.conv2d(ctx.encrypt(ctx.encode(img), ENC_SEED), layer, 5)
    assert np.abs(ctx.decrypt(out) - golden["cfg1/slots"]).max() < TOL


def test_conv_cfg5_three_layer_stack(oracle, golden):
    """cfg5: three 3x3 16->16 layers, one rescale each (13 -> 12 -> 11 -> 10 primes)."""
    p = pair(oracle, "cfg3")  # cfg5 shares cfg3's parameters
    x, _ = oracle.make_inputs(16, 32, 3, 16, 1003, 0, 0)
    ct = p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + 1)
    for li, sf in enumerate((2003, 2004, 2005)):
        _, filt = oracle.make_inputs(16, 32, 3, 16, 0, sf, 1)
        layer = p.ctx.conv_layer(16, 16, 32, 3, filt, level=ct.level)
        p.ctx.gen_galois_keys(layer.steps())
        ct = p.ctx.conv2d(ct, layer, (2, 3, 1)[li])
        assert ct.level == p.top - 1 - li
        err = np.abs(p.ctx.decrypt(ct) - golden[f"cfg5/out{li}"]).max()
        assert err < TOL, (li, err)


def test_conv_cfg5_three_layer_stack_fused(oracle, golden):
    """cfg5 through the fused schedule at levels 12, 11, 10 (digit counts 7, 6, 6)."""
    p = pair(oracle, "cfg3")
    x, _ = oracle.make_inputs(16, 32, 3, 16, 1003, 0, 0)
    ct = p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + 1)
    for li, sf in enumerate((2003, 2004, 2005)):
        _, filt = oracle.make_inputs(16, 32, 3, 16, 0, sf, 1)
        layer = p.ctx.conv_layer(16, 16, 32, 3, filt, level=ct.level)
        p.ctx.gen_galois_keys(layer.steps(5))
        ct = p.ctx.conv2d(ct, layer, 5)
        err = np.abs(p.ctx.decrypt(ct) - golden[f"cfg5/out{li}"]).max()
        assert err < TOL, (li, err)


@pytest.mark.parametrize("name", ["small_c4to2", "small_c4m4k1"])
@pytest.mark.parametrize("approach", [2, 3, 4, 5])
def test_conv_geometry_variants(oracle, golden, name, approach):
    """c_out < c_in and kappa = 1, packed into cfg1's 4096 slots."""
    p = pair(oracle, "cfg1")
    c, m, k, co, img, filt = conv_case(oracle, golden, name)
    # embed a 4-channel 4x4 image into 4096 slots by duplication (pack, d = 256)
    s = p.ctx.slots
    slots = np.tile(img, s // img.size)
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    ct = p.ctx.encrypt(p.ctx.encode(slots), ENC_SEED)
    out = p.ctx.decrypt(p.ctx.conv2d(ct, layer, approach))
    want = oracle.emu_conv_slots(c, m, k, co, s, img, filt, 2)
    assert np.abs(out - want).max() < TOL
    assert np.array_equal(want[: 64], golden[f"{name}/slots"])  # oracle == reference at s = 64


def test_cfg2_decomposed_rotations(oracle, golden):
    """cfg2: rotations by 1..127 through power-of-two keys only, positive vs
    signed decomposition (reference rot.cpp:21-46, :131-156)."""
    from paper_2306_09189_b200 import decompose
    p = pair(oracle, "cfg2")
    s = p.ctx.slots
    pow2 = [1 << i for i in range(8)]
    p.ctx.gen_galois_keys(pow2 + [-x for x in pow2])
    z = rnd(s, 9)
    ct = p.ctx.encrypt(p.ctx.encode(z), ENC_SEED)
    for k in (1, 5, 63, 96, 127):
        for strat in (0, 1):
            out = p.ctx.rotate_decomposed(ct, k, strat)
            assert np.abs(p.ctx.decrypt(out) - np.roll(z, -k)).max() < TOL
    # residues of the signed path equal sequential golden-model rotations
    ctr = p.ck.encrypt(p.ck.encode(z, p.ck.scale, p.top), p.top, ENC_SEED)
    cur = ctr
    for st in decompose(1, 127, s):
        cur = p.ck.rotate(cur, p.top, st)
    assert np.array_equal(p.ctx.rotate_decomposed(ct, 127, 1).residues(), cur)
    keyed = {strat: sum(len(decompose(strat, n, s)) for n in range(1, 128)) for strat in (0, 1)}
    assert keyed == {0: int(golden["plan_cfg2/strat0/total"][0]), 1: int(golden["plan_cfg2/strat1/total"][0])}


def test_cfg2_hoisted_stencil(oracle):
    p = pair(oracle, "cfg2")
    stencil = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1)]
    p.ctx.gen_galois_keys(stencil)
    z = rnd(p.ctx.slots, 10)
    ct = p.ctx.encrypt(p.ctx.encode(z), ENC_SEED)
    ctr = p.ck.encrypt(p.ck.encode(z, p.ck.scale, p.top), p.top, ENC_SEED)
    outs = p.ctx.rotate_hoisted(ct, stencil)
    ref = p.ck.rotate_hoisted(ctr, p.top, stencil)
    for i, k in enumerate(stencil):
        assert np.array_equal(outs[i].residues(), ref[i])
        assert np.abs(p.ctx.decrypt(outs[i]) - np.roll(z, -k)).max() < TOL


@pytest.mark.parametrize("name,approach,n", [("cfg1", 4, 5), ("cfg3", 3, 5), ("cfg3", 0, 5), ("cfg1", 5, 5),
                                             ("cfg3", 5, 5), ("cfg1", 5, 2), ("cfg1", 5, 3), ("cfg1", 5, 9),
                                             ("cfg1", 1, 5), ("cfg1", 2, 5), ("cfg3", 1, 3), ("cfg3", 2, 3),
                                             ("cfg1", 2, 10)])
def test_batched_conv_equals_single(oracle, golden, name, approach, n):
    """fhe_conv2d_batch (keys/plaintexts streamed once per batch) = per-ciphertext conv, bit for bit."""
    p = pair(oracle, name)
    c, m, k, co, img, filt = conv_case(oracle, golden, name)
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(np.roll(img, 37 * i)), ENC_SEED + i) for i in range(n)]
    outs = p.ctx.conv2d_batch(cts, layer, approach)
    for i, ct in enumerate(cts):
        assert np.array_equal(outs[i].residues(), p.ctx.conv2d(ct, layer, approach).residues())
    err = np.abs(p.ctx.decrypt(outs[0]) - golden[f"{name}/slots"]).max()
    assert err < TOL, err


@pytest.mark.parametrize("approach,chunk", [(5, 2), (3, 0)])
def test_host_pipelined_batch_equals_device_batch(oracle, golden, approach, chunk):
    """fhe_conv2d_batch_host (upload | conv | download overlapped) = per-ciphertext conv, bit for bit."""
    p = pair(oracle, "cfg1")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(np.roll(img, 11 * i)), ENC_SEED + i) for i in range(5)]
    host_in = np.stack([x.residues() for x in cts]).astype(np.uint64)
    out = p.ctx.conv2d_batch_host(host_in, len(cts), layer, approach, chunk=chunk)
    for i, ct in enumerate(cts):
        assert np.array_equal(out[i], p.ctx.conv2d(ct, layer, approach).residues())
    assert np.abs(p.ctx.decrypt(p.ctx.upload(out[0], p.top - 1)) - golden["cfg1/slots"]).max() < TOL


def test_host_pipelined_async_calls_chain(oracle, golden):
    """consecutive fhe_conv2d_batch_host_async calls pipeline into one another and
    produce the same residues as the synchronous call."""
    p = pair(oracle, "cfg1")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(np.roll(img, 5 * i)), ENC_SEED + i) for i in range(6)]
    host_in = np.stack([x.residues() for x in cts]).astype(np.uint64)
    want = p.ctx.conv2d_batch_host(host_in, 6, layer, 5, chunk=2)
    outs = [np.zeros_like(want) for _ in range(3)]
    for o in outs:
        p.ctx.conv2d_batch_host(host_in, 6, layer, 5, host_out=o, chunk=2, asynchronous=True)
    p.ctx.host_wait()
    for o in outs:
        assert np.array_equal(o, want)


def test_rotate_hoisted_batch_equals_single(p1):
    """fhe_rotate_hoisted_batch (keys shared by the ciphertexts of a batch) = per-ciphertext hoisting."""
    ks = [1, -1, 0, 32, -33, 1000]
    p1.ctx.gen_galois_keys([k for k in ks if k])
    rng = np.random.default_rng(21)
    cts = [p1.ctx.encrypt(p1.ctx.encode(rng.uniform(-1, 1, p1.ctx.slots)), ENC_SEED + i) for i in range(5)]
    outs = p1.ctx.rotate_hoisted_batch(cts, ks)
    for i, ct in enumerate(cts):
        single = p1.ctx.rotate_hoisted(ct, ks)
        for j in range(len(ks)):
            assert np.array_equal(outs[i][j].residues(), single[j].residues())


@pytest.mark.parametrize("name", ["ms_cfg1_c8", "ms_cfg1_c8to4", "ms_cfg1_c4to8"])
def test_multishard_conv_bit_exact_and_within_tolerance(oracle, golden, p1, name):
    """multi-shard image mode: t input / n_out output ciphertexts, bit-exact vs
    the golden model's ck_conv_shards, decrypted within 1e-6 of the reference's conv_image_shards."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    t = c * m * m // s
    layer = p1.ctx.conv_layer_shards(c, co, m, k, filt)
    assert layer.t == t and layer.n_out == golden[f"{name}/slots"].shape[0]
    p1.ctx.gen_galois_keys(layer.steps())
    cts = [p1.ctx.encrypt(p1.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(t)]
    outs = p1.ctx.conv2d_shards(cts, layer)
    ctr = np.stack([p1.ck.encrypt(p1.ck.encode(img[u * s:(u + 1) * s], p1.ck.scale, p1.top), p1.top, ENC_SEED + u)
                    for u in range(t)])
    ref, sc = p1.ck.conv_shards(ctr, p1.top, c, m, k, co, filt)
    for v, o in enumerate(outs):
        assert np.array_equal(o.residues(), ref[v])
        assert np.abs(p1.ctx.decrypt(o) - golden[f"{name}/slots"][v]).max() < TOL
    # two images at once = one at a time
    outs2 = p1.ctx.conv2d_shards(cts + cts[::-1], layer)
    for v in range(layer.n_out):
        assert np.array_equal(outs2[v].residues(), outs[v].residues())


def test_multishard_conv_cfg3(oracle, golden):
    """cfg3 parameters, 32 channels of 32x32 (t = 2 input, n_out = 2 output ciphertexts)."""
    p = pair(oracle, "cfg3")
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden["ms_cfg3_c32/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    layer = p.ctx.conv_layer_shards(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(layer.t)]
    outs = p.ctx.conv2d_shards(cts, layer)
    for v, o in enumerate(outs):
        assert np.abs(p.ctx.decrypt(o) - golden["ms_cfg3_c32/slots"][v]).max() < TOL


@pytest.mark.parametrize("name", ["cs_cfg1_c2m128", "cs_cfg1_c2to4m128"])
def test_channel_shard_conv_bit_exact_and_within_tolerance(oracle, golden, p1, name):
    """channel-shard mode (m^2 > slots): bit-exact vs the golden model's
    ck_conv_channel, decrypted within 1e-6 of the reference's conv_channel_shards."""
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    layer = p1.ctx.conv_layer_shards(c, co, m, k, filt)
    nin = c * m * m // s
    assert layer.t == nin and layer.n_out == golden[f"{name}/slots"].shape[0]
    p1.ctx.gen_galois_keys(layer.steps())
    cts = [p1.ctx.encrypt(p1.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(nin)]
    outs = p1.ctx.conv2d_shards(cts, layer)
    ctr = np.stack([p1.ck.encrypt(p1.ck.encode(img[u * s:(u + 1) * s], p1.ck.scale, p1.top), p1.top, ENC_SEED + u)
                    for u in range(nin)])
    ref, _ = p1.ck.conv_channel(ctr, p1.top, c, m, k, co, filt)
    for v, o in enumerate(outs):
        assert np.array_equal(o.residues(), ref[v])
        assert np.abs(p1.ctx.decrypt(o) - golden[f"{name}/slots"][v]).max() < TOL


def test_channel_shard_conv_cfg3_5x5(oracle, golden):
    """cfg3 parameters: one 256x256 channel (4 shards) -> 2 channels, 5x5 kernel (giants in two chunks)."""
    p = pair(oracle, "cfg3")
    c, m, k, co, si, sf, wk, s = (int(x) for x in golden["cs_cfg3_c1m256k5/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    layer = p.ctx.conv_layer_shards(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(layer.t)]
    outs = p.ctx.conv2d_shards(cts, layer)
    for v, o in enumerate(outs):
        assert np.abs(p.ctx.decrypt(o) - golden["cs_cfg3_c1m256k5/slots"][v]).max() < TOL


def _golden_slot_sum(ck, x, level, block):
    acc = x
    step = 1
    while step < block:
        acc = ck.add(acc, ck.rotate(acc, level, step), level)
        step *= 2
    return acc


def test_slot_sum_batch_bit_exact(oracle, golden, p1):
    """fhe_slot_sum_batch (each step one batched keyed rotation) = sequential golden-model
    rotate-and-add, and decrypts to the reference's slot_sum."""
    vec = np.random.default_rng(77).uniform(-1, 1, 4096)
    p1.ctx.gen_galois_keys([1 << i for i in range(12)])
    cts = [p1.ctx.encrypt(p1.ctx.encode(np.roll(vec, -i)), ENC_SEED + i) for i in range(3)]
    outs = p1.ctx.slot_sum_batch(cts, 64)
    for i, ct in enumerate(cts):
        ctr = p1.ck.encrypt(p1.ck.encode(np.roll(vec, -i), p1.ck.scale, p1.top), p1.top, ENC_SEED + i)
        assert np.array_equal(outs[i].residues(), _golden_slot_sum(p1.ck, ctr, p1.top, 64))
    assert np.abs(p1.ctx.decrypt(outs[0]) - golden["slot_sum/block64"]).max() < TOL


@pytest.mark.parametrize("name", ["lin_cfg1_c4m32", "lin_cfg1_c8m32", "lin_cfg1_c2m16", "lin_cfg1_c1m128"])
def test_linear_bit_exact_and_within_tolerance(oracle, golden, p1, name):
    """SURVEY §8(f) 3, the linear head: fhe_linear = the golden model's op sequence (masked products,
    slot sums, selection, bias) bit for bit, decrypted within 1e-6 of the reference's linear()."""
    c, m, s, no, si, t = (int(x) for x in golden[f"{name}/params"])
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    rng = np.random.default_rng(si)
    w = rng.uniform(-1, 1, no * c * m * m)
    b = rng.uniform(-1, 1, no)
    flat = img if img.size >= s else np.tile(img, s // img.size)
    chunks = [flat[u * s:(u + 1) * s] for u in range(t)]
    p1.ctx.gen_galois_keys([1 << i for i in range(12)])
    cts = [p1.ctx.encrypt(p1.ctx.encode(x), ENC_SEED + u) for u, x in enumerate(chunks)]
    out = p1.ctx.linear(cts, c, m, w, b)
    dec = p1.ctx.decrypt(out)
    # cfg1 scale 2^40 and up to 8192-term dot products (|y| ~ 30): the CKKS noise of the
    # summed products is held to 1e-6 relative to max(1, |y|); residues are bit-exact below
    want = golden[f"{name}/slots"]
    assert (np.abs(dec[:no] - want) / np.maximum(1.0, np.abs(want))).max() < TOL
    assert np.abs(dec[no:]).max() < TOL
    # golden model, the same op sequence
    ck, L = p1.ck, p1.top
    nin = c * m * m
    shards = [ck.encrypt(ck.encode(x, ck.scale, L), L, ENC_SEED + u) for u, x in enumerate(chunks)]
    sums = []
    for o in range(no):
        started = False
        for u in range(t):
            feat = np.arange(u * s, (u + 1) * s)
            wt = np.where(feat < nin, w.reshape(no, nin)[o][np.minimum(feat, nin - 1)], 0.0)
            if not wt.any() and started:
                continue
            x = ck.rescale(ck.mul_plain(shards[u], ck.encode(wt, float(ck.primes[L]), L), L), L)
            sums.append((o, _golden_slot_sum(ck, x, L - 1, s)))
            started = True
    acc = None
    for o in range(no):
        parts = [x for oo, x in sums if oo == o]
        total = parts[0]
        for x in parts[1:]:
            total = ck.add(total, x, L - 1)
        sel = np.zeros(s)
        sel[o] = 1.0
        y = ck.rescale(ck.mul_plain(total, ck.encode(sel, float(ck.primes[L - 1]), L - 1), L - 1), L - 1)
        acc = y if acc is None else ck.add(acc, y, L - 2)
    bias = np.zeros(s)
    bias[:no] = b
    ref = ck.add_plain(acc, ck.encode(bias, ck.scale, L - 2), L - 2)
    assert np.array_equal(out.residues(), ref)


def _golden_pool(ck, cts, level, c, m, s):
    """the golden model's pooling: three ck_lintrans stages (rotated masks), then the reference's
    consolidation / duplication rotations and adds."""
    block, bn = m * m, (m // 2) ** 2
    t = len(cts)
    rot = lambda v, k: np.roll(v, -k)

    def wmask(kk, ll):
        v = np.zeros(s)
        for b in range(s // block):
            for i in range(m - kk):
                v[b * block + i * m: b * block + i * m + (m - ll)] = 0.25
        return v
    aw = [0, 1, m, m + 1]
    pw = [wmask(0, 0), wmask(0, 1), wmask(1, 0), wmask(1, 1)]
    ah, ph, av, pv = [], [], [], []
    for i in range(m // 2):
        mk = np.zeros(s)
        mk[2 * i::m] = 1.0
        ah.append(i)
        ph.append(rot(mk, i))
        mv = np.zeros(s)
        for b in range(s // block):
            mv[b * block + 2 * i * m: b * block + 2 * i * m + m // 2] = 1.0
        av.append(3 * i * m // 2)
        pv.append(rot(mv, 3 * i * m // 2))
    V = []
    for x in cts:
        w_ = ck.lintrans(x, level, aw, pw)
        h_ = ck.lintrans(w_, level - 1, ah, ph)
        V.append(ck.lintrans(h_, level - 2, av, pv))
    L = level - 3
    if t == 1:
        base = V[0]
        out = base
        for e in range(1, 4):
            out = ck.add(out, ck.rotate(base, L, -e * bn), L)
        return [out]
    if t == 2:
        sm = ck.add(V[0], ck.rotate(V[1], L, -2 * bn), L)
        return [ck.add(sm, ck.rotate(sm, L, -bn), L)]
    res = []
    for w4 in range(t // 4):
        acc = V[4 * w4]
        for q in range(1, 4):
            acc = ck.add(acc, ck.rotate(V[4 * w4 + q], L, -q * bn), L)
        res.append(acc)
    return res


@pytest.mark.parametrize("name", ["pool_cfg1_c4m32", "pool_cfg1_c8m32", "pool_cfg1_c16m32"])
def test_pool_bit_exact_and_within_tolerance(oracle, golden, p1, name):
    """SURVEY §8(f) 2, 2x2 average pooling: bit-exact vs the golden model's staged pooling,
    decrypted within 1e-6 of the reference's pool() shards, same packing metadata."""
    c, m, s, si = (int(x) for x in golden[f"{name}/params"])
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    t = c * m * m // s
    bn = (m // 2) ** 2
    steps = [0, 1, m, m + 1] + list(range(m // 2)) + [3 * j * m // 2 for j in range(m // 2)] + \
            [-e * bn for e in range(1, 4)]
    p1.ctx.gen_galois_keys(sorted({k for k in steps if k}))
    chunks = [img[u * s:(u + 1) * s] for u in range(t)]
    cts = [p1.ctx.encrypt(p1.ctx.encode(x), ENC_SEED + u) for u, x in enumerate(chunks)]
    outs, tau, rep, d = p1.ctx.pool(cts, c, m)
    meta = golden[f"{name}/meta"]
    assert len(outs) == int(meta[5]) and rep == int(meta[3]) and d == int(meta[2])
    assert np.array_equal(tau, golden[f"{name}/tau"].astype(np.int64))
    for u, o in enumerate(outs):
        assert np.abs(p1.ctx.decrypt(o) - golden[f"{name}/slots"][u]).max() < TOL
    ctr = [p1.ck.encrypt(p1.ck.encode(x, p1.ck.scale, p1.top), p1.top, ENC_SEED + u) for u, x in enumerate(chunks)]
    ref = _golden_pool(p1.ck, ctr, p1.top, c, m, s)
    for o, r in zip(outs, ref):
        assert np.array_equal(o.residues(), r)


DS = ["ds_cfg1_c2m128_pool", "ds_cfg1_c1m256_pool", "ds_cfg1_c1m128_pool", "ds_cfg2_c1m128_pool",
      "ds_cfg1_c2m32_pool", "ds_cfg1_c8m32_pool_sc", "ds_cfg1_c4m32_s2", "ds_cfg1_c16m32_s2",
      "ds_cfg1_c2m128_s2", "ds_cfg1_c1m256_s2"]


@pytest.mark.parametrize("name", DS)
def test_downsample_bit_exact_and_within_tolerance(oracle, golden, name):
    """SURVEY §8(f) 2, pool() / subsample_stride2() over channel shards, duplicated inputs and
    output scales: residues bit-exact vs the golden model running the same stages
    (oracle.downsample_restated over ck_lintrans_src / ck_rotate / ck_add), decrypted shards
    within 1e-6 of the reference's, same packing metadata (tau, rep, d, mode)."""
    c, m, s, window, osc, si = golden[f"{name}/params"]
    c, m, s, window, si, osc = int(c), int(m), int(s), int(window), int(si), float(osc)
    p = pair(oracle, "cfg1" if s == 4096 else "cfg2")
    assert p.ctx.slots == s
    img, _ = oracle.make_inputs(c, m, 1, 1, si, 0, 0)
    block = m * m
    d_in = s // (block * c) if block <= s and block * c < s else 1
    chunks = list(np.tile(img, d_in).reshape(-1, s))
    p.ctx.gen_galois_keys(oracle.downsample_steps(c, m, s, bool(window)))
    cts = [p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + u) for u, x in enumerate(chunks)]
    if osc == 1.0 and d_in == 1:
        fn = p.ctx.pool if window else p.ctx.subsample_stride2
        outs, tau, rep, d = fn(cts, c, m)
        mode = int(m * m // 4 > s)
    else:
        outs, tau, rep, d, mode = p.ctx.downsample(cts, c, m, d=d_in, window=bool(window), output_scale=osc)
    meta = golden[f"{name}/meta"]
    assert (len(outs), rep, d, mode) == (int(meta[5]), int(meta[3]), int(meta[2]), int(meta[4]))
    assert np.array_equal(tau, golden[f"{name}/tau"].astype(np.int64))
    for u, o in enumerate(outs):
        assert o.level == p.top - (3 if window else 2)
        assert np.abs(p.ctx.decrypt(o) - golden[f"{name}/slots"][u]).max() < TOL
    ctr = [(p.ck.encrypt(p.ck.encode(x, p.ck.scale, p.top), p.top, ENC_SEED + u), p.top)
           for u, x in enumerate(chunks)]
    ref, *_ = oracle.downsample_restated(oracle.CkksOps(p.ck), ctr, c, m, s, bool(window), osc, d_in=d_in)
    for o, r in zip(outs, ref):
        assert np.array_equal(o.residues(), r[0])


def test_downsample_errors(p1):
    """the reference's exception texts (pool.cpp:231-306, pack.cpp:54-70)."""
    from paper_2306_09189_b200 import FheError
    ct = p1.ctx.encrypt(p1.ctx.encode(rnd(p1.ctx.slots, 3)), ENC_SEED)
    with pytest.raises(FheError, match="cannot pool a 1x1 channel"):
        p1.ctx.pool([ct], 4, 1)
    with pytest.raises(FheError, match="cannot subsample a 1x1 channel"):
        p1.ctx.subsample_stride2([ct], 4, 1)
    with pytest.raises(FheError, match="duplicated multi-shard image"):
        p1.ctx.downsample([ct, ct], 8, 32, d=2)
    with pytest.raises(FheError, match="metadata mismatch"):
        p1.ctx.pool([ct], 8, 32)
    with pytest.raises(FheError, match="dimensions must be powers of two"):
        p1.ctx.pool([ct], 3, 32)


# ------------------------------------------------------------ ct x ct, Chebyshev

CHEB = ["cheb_cfg3_gelu27_pre", "cheb_cfg3_gelu59_raw", "cheb_cfg3_relu27_raw", "cheb_cfg3_relu16_raw",
        "cheb_cfg1_gelu7_raw", "cheb_cfg1_identity", "cheb_cfg1_const"]
# golden-model composition is CPU-heavy at cfg3; these are also checked residue for residue
CHEB_BIT_EXACT = {"cheb_cfg3_gelu27_pre", "cheb_cfg1_gelu7_raw", "cheb_cfg1_identity", "cheb_cfg1_const"}


def cheb_input(golden, name):
    deg, bound, pre, level, s, seed = golden[f"{name}/params"]
    x = np.random.default_rng(int(seed)).uniform(-bound, bound, int(s))
    if pre:
        x = x / bound
    assert np.array_equal(np.array([x.sum(), np.abs(x).sum()]), golden[f"{name}/x_sum"])
    return x, int(deg), float(bound), bool(pre), int(level)


def test_mul_relin_bit_exact(p1):
    """fhe_mul (tensor, relinearisation with the s^2 key, rescale) = ck_mul_ct; operands at
    different levels are first brought to the common level (Engine::mul_ct's min level)."""
    ctx, ck, L = p1.ctx, p1.ck, p1.top
    ctx.gen_relin_key()
    a, b = rnd(ctx.slots, 31), rnd(ctx.slots, 32)
    ca = ctx.encrypt(ctx.encode(a), ENC_SEED)
    cb = ctx.encrypt(ctx.encode(b, level=L - 1), ENC_SEED + 1)
    out = ctx.mul(ca, cb)
    assert out.level == L - 2
    want = ck.mul_ct(ca.residues()[:, :L], cb.residues(), L - 1)
    assert np.array_equal(out.residues(), want)
    assert np.abs(ctx.decrypt(out) - a * b).max() < TOL
    sq = ctx.mul(out, out)  # a second level: keys and scales compose
    assert np.array_equal(sq.residues(), ck.mul_ct(want, want, L - 2))
    assert np.abs(ctx.decrypt(sq) - (a * b) ** 2).max() < 1e-5


def test_scalar_ops_bit_exact(p1):
    """fhe_add_scalar / fhe_mul_scalar: the constant polynomial round(k * scale) (its NTT rows are
    the constant), added to c0 / multiplied in and rescaled with the scale kept exactly."""
    ctx, ck, L = p1.ctx, p1.ck, p1.top
    a = rnd(ctx.slots, 41)
    ca = ctx.encrypt(ctx.encode(a), ENC_SEED)

    def rows(v, lv):
        iv = int(np.rint(v))
        return np.stack([np.full(ck.N, iv % int(ck.primes[i]), dtype=np.uint64) for i in range(lv + 1)])

    s1 = ctx.add_scalar(ca, -0.375)
    assert np.array_equal(s1.residues(), ck.add_plain(ca.residues(), rows(-0.375 * ctx.scale, L), L))
    assert np.abs(ctx.decrypt(s1) - (a - 0.375)).max() < TOL
    m1 = ctx.mul_scalar(ca, -2.5)
    assert m1.level == L - 1 and m1.scale == ctx.scale
    want = ck.rescale(ck.mul_plain(ca.residues(), rows(-2.5 * ctx.scale * float(ck.primes[L]) / ctx.scale, L), L), L)
    assert np.array_equal(m1.residues(), want)
    assert np.abs(ctx.decrypt(m1) - (-2.5 * a)).max() < TOL


def test_mul_requires_relin_key():
    from paper_2306_09189_b200 import Context, FheError
    ctx = Context.from_config("cfg1")
    ctx.keygen(KEY_SEED)
    ct = ctx.encrypt(ctx.encode(rnd(ctx.slots, 1)), ENC_SEED)
    with pytest.raises(FheError, match="relinearisation key"):
        ctx.mul(ct, ct)


@pytest.mark.parametrize("name", CHEB)
def test_chebyshev_matches_reference(oracle, golden, name):
    """fhe_eval_chebyshev decrypts within 1e-6 of the reference's eval_chebyshev slots
    (act.cpp:151-162), lands on the reference's output level with the same op counts, and
    (CHEB_BIT_EXACT) equals the golden model's composition residue for residue."""
    p = pair(oracle, "cfg3" if "cfg3" in name else "cfg1")
    x, deg, bound, pre, level = cheb_input(golden, name)
    co = golden[f"{name}/coeffs"]
    p.ctx.gen_relin_key()
    ct = p.ctx.encrypt(p.ctx.encode(x, level=level), ENC_SEED)
    p.ctx.ledger_reset()
    y = p.ctx.eval_chebyshev(ct, co, bound, pre)
    lg = p.ctx.ledger()
    want_level, want_depth = golden[f"{name}/meta"]
    assert y.level == want_level
    assert abs(y.scale - p.ctx.scale) <= 1e-9 * p.ctx.scale
    dec = p.ctx.decrypt(y)
    want = golden[f"{name}/slots"]
    assert np.abs(dec[: want.size] - want).max() < TOL
    assert np.abs(dec - oracle.cheb_eval(co, bound, x * (bound if pre else 1.0))).max() < TOL
    ref_ledger = golden[f"{name}/ledger"]
    assert (lg["ct_pt_mults"], lg["ct_ct_mults"], lg["adds"], lg["max_depth_consumed"]) == \
        (ref_ledger[3], ref_ledger[4], ref_ledger[5], ref_ledger[7])
    if name in CHEB_BIT_EXACT:
        ck = p.ck
        ctr = ck.encrypt(ck.encode(x, ck.scale, level), level, ENC_SEED)
        out, lv, _ = ck.eval_chebyshev(ctr, level, ck.scale, co, bound, pre)
        assert lv == y.level
        assert np.array_equal(y.residues(), out)


def test_chebyshev_insufficient_level(oracle, golden):
    from paper_2306_09189_b200 import FheError
    p = pair(oracle, "cfg3")
    p.ctx.gen_relin_key()
    ct = p.ctx.encrypt(p.ctx.encode(np.full(p.ctx.slots, 0.1), level=3), ENC_SEED)
    with pytest.raises(FheError, match=bytes(golden["cheb_level_error"]).decode()):
        p.ctx.eval_chebyshev(ct, golden["cheb_cfg3_gelu27_pre/coeffs"], 10.0, True)


def test_downsample_missing_key_is_an_error_and_leaks_nothing():
    """a pool without its Galois keys fails with FHE_E_NOKEY; the intermediate ciphertexts are
    freed (the context's device pool returns to its level), and the context stays usable."""
    from paper_2306_09189_b200 import CONFIGS, Context, FheError
    ctx = Context(**CONFIGS["cfg1"])
    ctx.keygen(7)
    ct = ctx.encrypt(ctx.encode(rnd(ctx.slots, 4)), ENC_SEED)
    with pytest.raises(FheError, match="key"):
        ctx.pool([ct], 4, 32)
    ctx.gen_galois_keys([1])
    assert np.abs(ctx.decrypt(ctx.rotate(ct, 1)) - np.roll(ctx.decrypt(ct), -1)).max() < 1e-6


@pytest.mark.parametrize("name", ["pc_cfg1_c4m32", "pc_cfg1_c8m32", "pc_cfg1_c16m32", "pc_cfg1_c2m32"])
def test_packed_conv_after_pool_bit_exact(oracle, golden, p1, name):
    """convolve() of a pooled map (fhe_conv_layer_create_packed: tau, rep, duplication):
    residues bit-exact vs the golden model's ck_conv_packed on the same pooled ciphertexts,
    decrypted within 1e-6 of the reference's convolve(pool(pack(img)))."""
    c, m, s, kap, co, si, sf = (int(x) for x in golden[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, kap, co, si, sf, 0)
    block = m * m
    d_in = s // (block * c) if block * c < s else 1
    chunks = list(np.tile(img, d_in).reshape(-1, s))
    p1.ctx.gen_galois_keys(oracle.downsample_steps(c, m, s, True))
    cts = [p1.ctx.encrypt(p1.ctx.encode(x), ENC_SEED + u) for u, x in enumerate(chunks)]
    pooled, tau, rep, d, mode = p1.ctx.downsample(cts, c, m, d=d_in)
    layer = p1.ctx.conv_layer_packed(c, co, m // 2, kap, filt, t=len(pooled), tau=tau, rep=rep, d=d,
                                     level=pooled[0].level)
    p1.ctx.gen_galois_keys(layer.steps())
    outs = p1.ctx.conv2d_shards(pooled, layer)
    want = golden[f"{name}/slots"]
    assert len(outs) == want.shape[0] and layer.d_out == int(golden[f"{name}/meta"][2])
    for u, o in enumerate(outs):
        assert np.abs(p1.ctx.decrypt(o) - want[u]).max() < TOL
    ref, _ = p1.ck.conv_packed(np.stack([x.residues() for x in pooled]), pooled[0].level, c, m // 2, kap, co, filt,
                               tau, rep, d)
    for o, r in zip(outs, ref):
        assert np.array_equal(o.residues(), r)


@pytest.mark.parametrize("strat", [0, 1, 2])
def test_execute_schedule_matches_reference_plan(oracle, golden, strat):
    """plan_rotations + execute_schedule (rot.cpp:96-156) on the cfg2 stencil (m = 32, one
    same-source group): the reference's keyed-step total and grouping, outputs equal the
    slot rotations, residues equal the golden model's sequential rotations."""
    p = pair(oracle, "cfg2")
    s = p.ctx.slots
    stencil = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1)]
    pow2 = [1 << i for i in range(14)]
    p.ctx.gen_galois_keys(pow2 + [-x for x in pow2] + [a for a in stencil if a])
    z = rnd(s, 31)
    ct = p.ctx.encrypt(p.ctx.encode(z), ENC_SEED)
    outs, tot, groups, hoisted = p.ctx.execute_schedule(ct, stencil, [0] + [1] * 8, strat)
    assert tot == int(golden[f"plan_stencil/strat{strat}/total"][0])
    assert (groups, hoisted) == (1, 1)
    for a, o in zip(stencil, outs):
        assert np.abs(p.ctx.decrypt(o) - np.roll(z, -a)).max() < TOL
    from paper_2306_09189_b200 import decompose
    ctr = p.ck.encrypt(p.ck.encode(z, p.ck.scale, p.top), p.top, ENC_SEED)
    a = stencil[0]
    steps = [a % s] if strat == 2 else decompose(strat, a % s, s)
    cur = ctr
    for st in steps:
        if st % s:
            cur = p.ck.rotate(cur, p.top, st)
    assert np.array_equal(outs[0].residues(), cur)
    # without same-source flags every request is its own sequential group
    outs2, tot2, groups2, hoisted2 = p.ctx.execute_schedule(ct, stencil, [0] * 9, strat)
    assert (tot2, groups2, hoisted2) == (tot, 9, 0)
    assert np.array_equal(outs2[0].residues(), cur)


def test_linear_missing_key_is_an_error():
    """linear() without its slot-sum keys fails with the missing-key error (products freed)."""
    from paper_2306_09189_b200 import CONFIGS, Context, FheError
    ctx = Context(**CONFIGS["cfg1"])
    ctx.keygen(7)
    ct = ctx.encrypt(ctx.encode(rnd(ctx.slots, 5)), ENC_SEED)
    with pytest.raises(FheError, match="key"):
        ctx.linear([ct], 4, 32, rnd(2 * 4096, 6), rnd(2, 7))


@pytest.mark.parametrize("c,m,k", [(16, 16, 7), (4, 32, 7), (1, 64, 9)])
def test_conv_large_kernels_fused_schedule(oracle, c, m, k):
    """kernels up to 9x9 and c kappa beyond one fused launch (16 x 7 = 112 baby steps run in
    two launches per giant chunk): the default schedule is bit-exact with the golden model's
    fused BSGS (plan 5), batched = single, decrypted within 1e-6 of a float64 conv."""
    p = pair(oracle, "cfg1")
    img, filt = oracle.make_inputs(c, m, k, c, 7000 + k, 8000 + k, 0)
    layer = p.ctx.conv_layer(c, c, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps(0))
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED)
    out = p.ctx.conv2d(ct, layer, 0)
    outs = p.ctx.conv2d_batch([ct, ct, ct], layer, 0)
    x = img.reshape(c, m, m)
    w = filt.reshape(c, c, k, k)
    h = k // 2
    xp = np.pad(x, ((0, 0), (h, h), (h, h)))
    ref = np.zeros((c, m, m))
    for r in range(k):
        for s in range(k):
            ref += np.einsum("fg,fij->gij", w[:, :, r, s], xp[:, r:r + m, s:s + m])
    assert np.abs(p.ctx.decrypt(out)[: c * m * m] - ref.ravel()).max() < TOL
    ctr = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, ENC_SEED)
    gold, _ = p.ck.conv(ctr, p.top, c, m, k, c, filt, 5)
    assert np.array_equal(out.residues(), gold)
    for o in outs:
        assert np.array_equal(o.residues(), gold)


def test_channel_shard_conv_many_input_channels(oracle):
    """channel-shard conv whose baby steps per output shard exceed one fused launch
    (16 input channels x 3 source shards x 3 column shifts = 144): chunked launches,
    bit-exact vs the golden model, decrypted within 1e-6 of a float64 conv."""
    p = pair(oracle, "cfg1")
    c, co, m, k = 16, 1, 128, 3
    img, filt = oracle.make_inputs(c, m, k, co, 7100, 8100, 0)
    layer = p.ctx.conv_layer_shards(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps())
    s = p.ctx.slots
    chunks = list(img.reshape(-1, s))
    cts = [p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + u) for u, x in enumerate(chunks)]
    outs = p.ctx.conv2d_shards(cts, layer)
    x = img.reshape(c, m, m)
    w = filt.reshape(c, co, k, k)
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    ref = sum(np.einsum("fg,fij->gij", w[:, :, r, t], xp[:, r:r + m, t:t + m]) for r in range(k) for t in range(k))
    got = np.concatenate([p.ctx.decrypt(o) for o in outs])
    assert np.abs(got - ref.ravel()).max() < TOL
    ctr = np.stack([p.ck.encrypt(p.ck.encode(x_, p.ck.scale, p.top), p.top, ENC_SEED + u)
                    for u, x_ in enumerate(chunks)])
    gold, _ = p.ck.conv_channel(ctr, p.top, c, m, k, co, filt)
    for o, g in zip(outs, gold):
        assert np.array_equal(o.residues(), g)


def test_new_entry_points_reject_bad_arguments(p1):
    """error texts of the packed conv, the feature-map linear and the schedule executor."""
    from paper_2306_09189_b200 import FheError
    s = p1.ctx.slots
    w = rnd(4 * 4 * 9, 1)
    with pytest.raises(FheError, match="tau is not a permutation"):
        p1.ctx.conv_layer_packed(4, 4, 32, 3, w, t=1, tau=[0, 0, 1, 2])
    with pytest.raises(FheError, match="metadata mismatch"):
        p1.ctx.conv_layer_packed(4, 4, 32, 3, w, t=2)
    with pytest.raises(FheError, match="duplicated multi-shard image"):
        p1.ctx.conv_layer_packed(4, 4, 16, 3, w, t=2, d=2)
    with pytest.raises(FheError, match="kernel size must be odd"):
        p1.ctx.conv_layer_packed(4, 4, 32, 2, rnd(4 * 4 * 4, 1))
    ct = p1.ctx.encrypt(p1.ctx.encode(rnd(s, 2)), ENC_SEED)
    fm = np.full((1, s), -1, dtype=np.int64)
    fm[0, :8] = np.arange(8) + 100
    with pytest.raises(FheError, match="in_features does not match"):
        p1.ctx.linear_features([ct], fm, rnd(2 * 8, 3), rnd(2, 4))
    with pytest.raises(FheError, match="unknown decomposition strategy"):
        p1.ctx.execute_schedule(ct, [1, 2], [0, 1], 7)
