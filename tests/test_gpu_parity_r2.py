"""GPU parity of the configurations that are actually timed, the conv boundary's
bias / output_scale, and the regressions the round-1 review found.

* cfg5 (BASELINE: three 3x3 16->16 layers at levels 12 / 11 / 10, batch of 32):
  residues of every layer bit-exact with the golden model, for the single
  path and for members of the batch-32 path (reference conv_plan applied three
  times, conv.cpp:266-271);
* cfg3 approach 5 at batch 16 through fhe_conv2d_batch_into under CUDA-graph
  capture and replay (the bench's timed step);
* cfg3 hoisted rotations at batch 16 (fhe_rotate_hoisted_batch_into, the bench's
  hoisted-rotation metric; reference rotate_many emu.cpp:39-54);
* bias + output_scale on the conv layer (conv.hpp:46-68, bias_plain conv.cpp:87-94,
  conv_channel_shards conv.cpp:344): residues equal the golden conv followed by
  add_plain of the bias plaintext; decrypted within 1e-6 of the reference's slots
  (tests/golden/golden_bias.npz, tests/golden/make_golden_bias.py);
* keygen after a captured conv graph (graphs embed key addresses).
Tolerance: 1e-6 absolute on decrypted slots; residues bit-exact."""
import os

import numpy as np
import pytest

from test_gpu_parity import ENC_SEED, KEY_SEED, TOL, conv_case, pair

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gbias():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_bias.npz")))


def cfg5_inputs(oracle, n):
    x, _ = oracle.make_inputs(16, 32, 3, 16, 1003, 0, 0)
    filts = [oracle.make_inputs(16, 32, 3, 16, 0, sf, 1)[1] for sf in (2003, 2004, 2005)]
    imgs = [np.roll(x, 97 * i) for i in range(n)]
    return imgs, filts


def golden_chain(p, img, seed, filts, plan):
    """the golden model's three-layer cfg5 chain (its own residues at every layer)"""
    ct = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, seed)
    outs, lv = [], p.top
    for f in filts:
        ct, _ = p.ck.conv(ct, lv, 16, 32, 3, 16, f, plan)
        lv -= 1
        outs.append(ct)
    return outs


@pytest.mark.parametrize("approach", [5, 2])
def test_cfg5_single_path_residues_every_layer(oracle, golden, approach):
    p = pair(oracle, "cfg3")
    (img,), filts = cfg5_inputs(oracle, 1)
    want = golden_chain(p, img, ENC_SEED + 1, filts, approach)
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED + 1)
    for li, f in enumerate(filts):
        layer = p.ctx.conv_layer(16, 16, 32, 3, f, level=ct.level)
        p.ctx.gen_galois_keys(layer.steps())
        ct = p.ctx.conv2d(ct, layer, approach)
        assert ct.level == p.top - 1 - li
        assert np.array_equal(ct.residues(), want[li]), f"layer {li}"
        assert np.abs(p.ctx.decrypt(ct) - golden[f"cfg5/out{li}"]).max() < TOL


def test_cfg5_batch32_members_residues_every_layer(oracle, golden):
    """the bench's cfg5 workload: 32 ciphertexts through three layers by fhe_conv2d_batch_into
    (approach 0 -> the fused schedule), members 0, 13 and 31 bit-exact at every layer"""
    p = pair(oracle, "cfg3")
    imgs, filts = cfg5_inputs(oracle, 32)
    cts = [p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + 100 + i) for i, x in enumerate(imgs)]
    layers = []
    lv = p.top
    for f in filts:
        ly = p.ctx.conv_layer(16, 16, 32, 3, f, level=lv)
        p.ctx.gen_galois_keys(ly.steps())
        layers.append(ly)
        lv -= 1
    outs = []
    cur = cts
    for ly in layers:
        nxt = [p.ctx.encrypt(p.ctx.encode(np.zeros(8), level=ly.level - 1), 1) for _ in cur]
        p.ctx.conv2d_batch_into(cur, ly, 0, nxt)
        outs.append(nxt)
        cur = nxt
    for i in (0, 13, 31):
        want = golden_chain(p, imgs[i], ENC_SEED + 100 + i, filts, 5)
        for li in range(3):
            assert np.array_equal(outs[li][i].residues(), want[li]), (i, li)
    for li in range(3):
        assert np.abs(p.ctx.decrypt(outs[li][0]) - golden[f"cfg5/out{li}"]).max() < TOL


def test_cfg3_fused_batch16_graph_capture_and_replay_bit_exact(oracle, golden):
    """the headline step: 16 ciphertexts, approach 5, fhe_conv2d_batch_into captured into a CUDA
    graph on the first call and replayed on the second; members 0, 7, 15 vs the golden model"""
    p = pair(oracle, "cfg3")
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg3")
    layer = p.ctx.conv_layer(c, co, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps(5))
    imgs = [np.roll(img, 41 * i) for i in range(16)]
    cts = [p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + 200 + i) for i, x in enumerate(imgs)]
    outs = [p.ctx.encrypt(p.ctx.encode(np.zeros(8), level=p.top - 1), 1) for _ in cts]
    p.ctx.conv2d_batch_into(cts, layer, 5, outs)  # capture + launch
    first = [o.residues() for o in outs]
    p.ctx.ledger_reset()
    p.ctx.conv2d_batch_into(cts, layer, 5, outs)  # replay
    lg = p.ctx.ledger()
    assert lg["distinct_amounts"] == len(layer.steps(5)) + 1  # the replay re-records its amounts (+ 0)
    for i in (0, 7, 15):
        ctr = p.ck.encrypt(p.ck.encode(imgs[i], p.ck.scale, p.top), p.top, ENC_SEED + 200 + i)
        ref, _ = p.ck.conv(ctr, p.top, c, m, k, co, filt, 5)
        assert np.array_equal(first[i], ref), i
        assert np.array_equal(outs[i].residues(), ref), i
    assert np.abs(p.ctx.decrypt(outs[0]) - golden["cfg3/slots"]).max() < TOL


def test_cfg3_hoisted_rotation_batch16_bit_exact(oracle):
    """the bench's hoisted-rotation metric: the 8 stencil shifts (m = 32) of 16 ciphertexts from one
    ModUp each (fhe_rotate_hoisted_batch_into), members 0 and 15 vs the golden model"""
    p = pair(oracle, "cfg3")
    ks = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
    p.ctx.gen_galois_keys(ks)
    rng = np.random.default_rng(31)
    zs = [rng.uniform(-1, 1, p.ctx.slots) for _ in range(16)]
    cts = [p.ctx.encrypt(p.ctx.encode(z), ENC_SEED + 300 + i) for i, z in enumerate(zs)]
    outs = [p.ctx.encrypt(p.ctx.encode(np.zeros(8)), 1) for _ in range(16 * len(ks))]
    p.ctx.rotate_hoisted_batch_into(cts, ks, outs)
    for i in (0, 15):
        ctr = p.ck.encrypt(p.ck.encode(zs[i], p.ck.scale, p.top), p.top, ENC_SEED + 300 + i)
        ref = p.ck.rotate_hoisted(ctr, p.top, ks)
        for j, kk in enumerate(ks):
            o = outs[i * len(ks) + j]
            assert np.array_equal(o.residues(), ref[j]), (i, kk)
        assert np.abs(p.ctx.decrypt(outs[i * len(ks)]) - np.roll(zs[i], -ks[0])).max() < TOL


def test_cfg2_hoisted_rotation_batch40_gathered_inputs_bit_exact(oracle):
    """batches of >= 32 ciphertexts gather their inputs through a device pointer table
    (k_gather_ptrs, one launch): BASELINE cfg2's building block (one batched keyed rotation of all
    ciphertexts, power-of-two keys) plus an identity amount, members 0 / 17 / 39 vs the golden model"""
    p = pair(oracle, "cfg2")
    ks = [4, 0, -16]
    p.ctx.gen_galois_keys([k for k in ks if k])
    rng = np.random.default_rng(47)
    n = 40
    zs = [rng.uniform(-1, 1, p.ctx.slots) for _ in range(n)]
    cts = [p.ctx.encrypt(p.ctx.encode(z), ENC_SEED + 700 + i) for i, z in enumerate(zs)]
    outs = [p.ctx.encrypt(p.ctx.encode(np.zeros(8)), 1) for _ in range(n * len(ks))]
    p.ctx.rotate_hoisted_batch_into(cts, ks, outs)
    for i in (0, 17, 39):
        ctr = p.ck.encrypt(p.ck.encode(zs[i], p.ck.scale, p.top), p.top, ENC_SEED + 700 + i)
        ref = p.ck.rotate_hoisted(ctr, p.top, ks)
        for j, kk in enumerate(ks):
            assert np.array_equal(outs[i * len(ks) + j].residues(), ref[j]), (i, kk)
        assert np.abs(p.ctx.decrypt(outs[i * len(ks)]) - np.roll(zs[i], -ks[0])).max() < TOL


# ------------------------------------------------------------------ bias / output_scale

def bias_case(oracle, gb, name):
    c, m, k, co, si, sf, wk, s, plan, bs = (int(x) for x in gb[f"{name}/params"])
    img, filt = oracle.make_inputs(c, m, k, co, si, sf, wk)
    return c, m, k, co, s, plan, img, filt, gb[f"{name}/bias"], float(gb[f"{name}/output_scale"][0])


def golden_bias_add(p, outs, sc, bias_vecs, level):
    """the golden model's conv output + add_plain(bias plaintext at the output level and scale)"""
    return [p.ck.add_plain(o, p.ck.encode(v, sc, level), level) for o, v in zip(outs, bias_vecs)]


def image_bias_vecs(bias, osc, c_out, m, s, n_out):
    """ImageConv::bias_plain (conv.cpp:87-94) for each output shard v"""
    block, z = m * m, s // (m * m)
    return [np.repeat(np.array([bias[(v * z + b) % c_out] * osc for b in range(z)]), block) for v in range(n_out)]


@pytest.mark.parametrize("name,approaches", [("bias_cfg1_a2", (2, 5)), ("bias_cfg1_a1", (1, 3))])
def test_conv_bias_output_scale_cfg1(oracle, gbias, name, approaches):
    p = pair(oracle, "cfg1")
    c, m, k, co, s, plan, img, filt, bias, osc = bias_case(oracle, gbias, name)
    layer = p.ctx.conv_layer(c, co, m, k, filt, bias=bias, output_scale=osc)
    p.ctx.gen_galois_keys(layer.steps())
    ct = p.ctx.encrypt(p.ctx.encode(img), ENC_SEED)
    ctr = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, ENC_SEED)
    for approach in approaches:
        out = p.ctx.conv2d(ct, layer, approach)
        ref, sc = p.ck.conv(ctr, p.top, c, m, k, co, filt * osc, approach)
        want = golden_bias_add(p, [ref], sc, image_bias_vecs(bias, osc, co, m, s, 1), p.top - 1)[0]
        assert np.array_equal(out.residues(), want), approach
        err = np.abs(p.ctx.decrypt(out) - gbias[f"{name}/slots"][0]).max()
        assert err < TOL, (approach, err)
    # batched path (fused kernel / paper batch) adds the same bias to every member
    outs = p.ctx.conv2d_batch([ct, ct, ct], layer, approaches[0])
    single = p.ctx.conv2d(ct, layer, approaches[0]).residues()
    for o in outs:
        assert np.array_equal(o.residues(), single)


def test_conv_bias_output_scale_cfg3_batch(oracle, gbias):
    p = pair(oracle, "cfg3")
    c, m, k, co, s, plan, img, filt, bias, osc = bias_case(oracle, gbias, "bias_cfg3_a2")
    layer = p.ctx.conv_layer(c, co, m, k, filt, bias=bias, output_scale=osc)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(img), ENC_SEED + i) for i in range(4)]
    outs = p.ctx.conv2d_batch(cts, layer, 5)
    ctr = p.ck.encrypt(p.ck.encode(img, p.ck.scale, p.top), p.top, ENC_SEED + 3)
    ref, sc = p.ck.conv(ctr, p.top, c, m, k, co, filt * osc, 5)
    want = golden_bias_add(p, [ref], sc, image_bias_vecs(bias, osc, co, m, s, 1), p.top - 1)[0]
    assert np.array_equal(outs[3].residues(), want)
    for o in outs:
        assert np.abs(p.ctx.decrypt(o) - gbias["bias_cfg3_a2/slots"][0]).max() < TOL
    two = p.ctx.conv2d(cts[0], layer, 2)
    assert np.abs(p.ctx.decrypt(two) - gbias["bias_cfg3_a2/slots"][0]).max() < TOL


@pytest.mark.parametrize("name", ["bias_ms_cfg1_c4to8", "bias_ms_cfg1_c8"])
def test_conv_bias_image_shards(oracle, gbias, name):
    p = pair(oracle, "cfg1")
    c, m, k, co, s, plan, img, filt, bias, osc = bias_case(oracle, gbias, name)
    t = max(1, c * m * m // s)
    layer = p.ctx.conv_layer_shards(c, co, m, k, filt, bias=bias, output_scale=osc)
    p.ctx.gen_galois_keys(layer.steps())
    cts = [p.ctx.encrypt(p.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(t)]
    outs = p.ctx.conv2d_shards(cts, layer)
    ctr = np.stack([p.ck.encrypt(p.ck.encode(img[u * s:(u + 1) * s], p.ck.scale, p.top), p.top, ENC_SEED + u)
                    for u in range(t)])
    ref, sc = p.ck.conv_shards(ctr, p.top, c, m, k, co, filt * osc)
    want = golden_bias_add(p, list(ref), sc, image_bias_vecs(bias, osc, co, m, s, len(ref)), p.top - 1)
    assert len(outs) == gbias[f"{name}/slots"].shape[0]
    for v, o in enumerate(outs):
        assert np.array_equal(o.residues(), want[v]), v
        assert np.abs(p.ctx.decrypt(o) - gbias[f"{name}/slots"][v]).max() < TOL


def test_conv_bias_channel_shards(oracle, gbias):
    p = pair(oracle, "cfg1")
    c, m, k, co, s, plan, img, filt, bias, osc = bias_case(oracle, gbias, "bias_cs_cfg1_c2m128")
    layer = p.ctx.conv_layer_shards(c, co, m, k, filt, bias=bias, output_scale=osc)
    p.ctx.gen_galois_keys(layer.steps())
    nin = c * m * m // s
    pc = m * m // s
    cts = [p.ctx.encrypt(p.ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(nin)]
    outs = p.ctx.conv2d_shards(cts, layer)
    ctr = np.stack([p.ck.encrypt(p.ck.encode(img[u * s:(u + 1) * s], p.ck.scale, p.top), p.top, ENC_SEED + u)
                    for u in range(nin)])
    ref, sc = p.ck.conv_channel(ctr, p.top, c, m, k, co, filt * osc)
    vecs = [np.full(s, bias[o // pc] * osc) for o in range(len(ref))]
    want = golden_bias_add(p, list(ref), sc, vecs, p.top - 1)
    for v, o in enumerate(outs):
        assert np.array_equal(o.residues(), want[v]), v
        assert np.abs(p.ctx.decrypt(o) - gbias["bias_cs_cfg1_c2m128/slots"][v]).max() < TOL


def test_conv_bias_size_checked(oracle, gbias):
    p = pair(oracle, "cfg1")
    c, m, k, co, s, plan, img, filt, bias, osc = bias_case(oracle, gbias, "bias_cfg1_a2")
    with pytest.raises(ValueError, match="bias size does not match output channels"):
        p.ctx.conv_layer(c, co, m, k, filt, bias=bias[:2])


# ------------------------------------------------------------------ regressions

def test_keygen_after_captured_conv_graph(oracle, golden):
    """a captured conv graph embeds the Galois-key addresses: keygen must drop it"""
    from paper_2306_09189_b200 import CONFIGS, Context
    c, m, k, co, img, filt = conv_case(oracle, golden, "cfg1")
    ctx = Context.from_config("cfg1")
    ctx.keygen(KEY_SEED)
    layer = ctx.conv_layer(c, co, m, k, filt)
    steps = layer.steps(5)
    ctx.gen_galois_keys(steps)
    cts = [ctx.encrypt(ctx.encode(img), ENC_SEED + i) for i in range(2)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in cts]
    ctx.conv2d_batch_into(cts, layer, 5, outs)
    ctx.conv2d_batch_into(cts, layer, 5, outs)  # replayed graph
    ctx.keygen(KEY_SEED + 1)
    ctx.gen_galois_keys(list(reversed(steps)) + [3, 5])  # other allocation order
    cts = [ctx.encrypt(ctx.encode(img), ENC_SEED + i) for i in range(2)]
    ctx.conv2d_batch_into(cts, layer, 5, outs)
    pr = CONFIGS["cfg1"]
    ck = oracle.CKKS(pr["log_n"], pr["q_bits"], pr["p_bits"], pr["log_scale"])
    ck.keygen(KEY_SEED + 1)
    top = ctx.max_level
    ctr = ck.encrypt(ck.encode(img, ck.scale, top), top, ENC_SEED + 1)
    ref, _ = ck.conv(ctr, top, c, m, k, co, filt, 5)
    assert np.array_equal(outs[1].residues(), ref)


def test_linear_head_plaintext_cache(oracle):
    """fhe_linear keeps the encoded weight / selection / bias plaintexts of a head (keyed by a hash
    of weights, bias, feature map, level and scale): a second call with the same head reuses them and
    gives identical residues; other weights, another bias or another input level miss the cache and
    give their own results (reference linear() dense.cpp:34-75 has no state to get stale)."""
    p = pair(oracle, "cfg1")
    rng = np.random.default_rng(91)
    c, m, no = 4, 32, 3
    p.ctx.gen_galois_keys([1 << i for i in range(12)])
    x = rng.uniform(-1, 1, p.ctx.slots)
    ct = p.ctx.encrypt(p.ctx.encode(x), ENC_SEED + 900)
    w1, b1 = rng.uniform(-1, 1, no * c * m * m), rng.uniform(-1, 1, no)
    w2, b2 = rng.uniform(-1, 1, no * c * m * m), rng.uniform(-1, 1, no)

    def want(w, b):
        return w.reshape(no, -1) @ x + b

    first = p.ctx.linear([ct], c, m, w1, b1)
    other = p.ctx.linear([ct], c, m, w2, b1)       # miss: other weights
    biased = p.ctx.linear([ct], c, m, w1, b2)      # miss: other bias
    again = p.ctx.linear([ct], c, m, w1, b1)       # hit
    assert np.array_equal(first.residues(), again.residues())
    for out, (w, b) in ((first, (w1, b1)), (other, (w2, b1)), (biased, (w1, b2)), (again, (w1, b1))):
        y = want(w, b)
        assert (np.abs(p.ctx.decrypt(out)[:no] - y) / np.maximum(1.0, np.abs(y))).max() < TOL
    # five more heads evict the first (4 kept); it is re-encoded and still right
    for i in range(5):
        p.ctx.linear([ct], c, m, rng.uniform(-1, 1, no * c * m * m), b1)
    back = p.ctx.linear([ct], c, m, w1, b1)
    assert np.array_equal(first.residues(), back.residues())
