"""GPU parity of channel-shard convs whose shards hold one or two image rows
(rows per shard = slots / m = 1 or 2: the reference's conv_channel_shards,
conv.cpp:273-362, with its reach check at :286 at the limit), at a small ring
(N = 2^12, 2048 slots) so the shard counts stay testable: m = 1024 (2 rows per
shard, 512 shards) bit-exact against the golden model's ck_conv_channel and
decrypted within 1e-6 of the reference restatement (emu_conv_channel_slots,
pinned to the reference in test_oracle_pins.py); m = 2048 (1 row per shard,
2048 shards: the row shifts kk m are whole-slot rotations, i.e. identities)
likewise."""
import numpy as np
import pytest

from test_gpu_parity import ENC_SEED, KEY_SEED, TOL

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

PARAMS = dict(log_n=12, q_bits=[60, 40, 40], p_bits=[60], log_scale=40)


@pytest.mark.parametrize("m,residues", [(1024, True), (2048, True)])
def test_single_and_double_row_channel_shards(oracle, m, residues):
    from paper_2306_09189_b200 import Context
    c, co, k = 1, 1, 3
    s = (1 << PARAMS["log_n"]) // 2
    img, filt = oracle.make_inputs(c, m, k, co, 31, 32, 0)
    ctx = Context(**PARAMS)
    ctx.keygen(KEY_SEED)
    layer = ctx.conv_layer_shards(c, co, m, k, filt)
    nin = c * m * m // s
    assert layer.t == nin and layer.n_out == co * m * m // s
    ctx.gen_galois_keys(layer.steps())
    cts = [ctx.encrypt(ctx.encode(img[u * s:(u + 1) * s]), ENC_SEED + u) for u in range(nin)]
    outs = ctx.conv2d_shards(cts, layer)
    want = oracle.emu_conv_channel_slots(c, m, k, co, s, img, filt)
    assert want.shape == (len(outs), s)
    err = max(np.abs(ctx.decrypt(o) - want[v]).max() for v, o in enumerate(outs))
    assert err < TOL, err
    if residues:
        ck = oracle.CKKS(PARAMS["log_n"], PARAMS["q_bits"], PARAMS["p_bits"], PARAMS["log_scale"])
        ck.keygen(KEY_SEED)
        top = ctx.max_level
        ctr = np.stack([ck.encrypt(ck.encode(img[u * s:(u + 1) * s], ck.scale, top), top, ENC_SEED + u)
                        for u in range(nin)])
        ref, _ = ck.conv_channel(ctr, top, c, m, k, co, filt)
        for v, o in enumerate(outs):
            assert np.array_equal(o.residues(), ref[v]), v
