"""GPU parity of the TMA-staged operand-form baby-step kernel (k_bsgs_tma, the default
for approach 5: FP64 products on rows q < 2^50, 30-bit limbs on the 60-bit rows) on the
shapes its staging has to get right:

* plaintext boxes across giant chunks (7x7 kernel: 7 giants = a 5-giant and a
  2-giant launch) and 5-giant launches (5x5);
* partial source groups (batches of 3, 5 and 6: the last group's box is shifted
  back inside the tensor) and single ciphertexts;
* the two fused kernels (k_bsgs_fused on plain rows, k_bsgs_tma on operand-form
  rows) give identical residues at cfg3, cfg1 (40-bit rows) and cfg4 (FHECONV_TMA=0
  selects k_bsgs_fused per context).

Residues are compared bit-exact with the golden model's approach-5 conv (reference
schedule: conv_plan conv.cpp:266-271 over the fused plaintexts conv.cpp:69-85).
Every case has a timeout: a staging bug shows up as an mbarrier that never completes."""
import os

import numpy as np
import pytest

from test_gpu_parity import ENC_SEED, pair

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.mark.parametrize("k", [3, 5, 7])
def test_tma_giant_chunks_and_partial_groups_bit_exact(oracle, k):
    p = pair(oracle, "cfg1")
    rng = np.random.default_rng(40 + k)
    c, m = 4, 32
    filt = rng.uniform(-1, 1, c * c * k * k)
    layer = p.ctx.conv_layer(c, c, m, k, filt)
    p.ctx.gen_galois_keys(layer.steps(5))
    imgs = [rng.uniform(-1, 1, c * m * m) for _ in range(6)]
    refs = {}
    for i in (0, 2, 4, 5):
        ctr = p.ck.encrypt(p.ck.encode(imgs[i], p.ck.scale, p.top), p.top, ENC_SEED + i)
        refs[i], _ = p.ck.conv(ctr, p.top, c, m, k, c, filt, 5)
    for B in (1, 3, 5, 6):
        cts = [p.ctx.encrypt(p.ctx.encode(imgs[i]), ENC_SEED + i) for i in range(B)]
        outs = [p.ctx.encrypt(p.ctx.encode(np.zeros(8), level=p.ctx.max_level - 1), 1) for _ in range(B)]
        p.ctx.conv2d_batch_into(cts, layer, 5, outs)
        for i in refs:
            if i < B:
                assert np.array_equal(outs[i].residues(), refs[i]), f"k={k} batch {B} member {i}"


@pytest.mark.parametrize("cfg,geo,B", [("cfg3", (16, 32, 3), 5), ("cfg1", (4, 32, 3), 6), ("cfg4", (8, 64, 5), 2)])
def test_fused_and_tma_kernels_identical(oracle, cfg, geo, B):
    from paper_2306_09189_b200 import Context
    rng = np.random.default_rng(5)
    c, m, k = geo
    filt = rng.uniform(-1, 1, c * c * k * k)
    imgs = [rng.uniform(-1, 1, c * m * m) for _ in range(B)]
    res = {}
    for name, env in (("fused", {"FHECONV_TMA": "0"}), ("tma", {})):
        old = {v: os.environ.get(v) for v in ("FHECONV_LIMB", "FHECONV_TMA")}
        for v in old:
            os.environ.pop(v, None)
        os.environ.update(env)
        try:
            ctx = Context.from_config(cfg)
        finally:
            for v, x in old.items():
                if x is None:
                    os.environ.pop(v, None)
                else:
                    os.environ[v] = x
        ctx.keygen(7)
        layer = ctx.conv_layer(c, c, m, k, filt)
        ctx.gen_galois_keys(layer.steps(5))
        cts = [ctx.encrypt(ctx.encode(x), ENC_SEED + i) for i, x in enumerate(imgs)]
        outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in imgs]
        ctx.conv2d_batch_into(cts, layer, 5, outs)
        single = ctx.conv2d(cts[0], layer, 5)
        res[name] = [o.residues() for o in outs] + [single.residues()]
        del ctx
    for a, b in zip(res["fused"], res["tma"]):
        assert np.array_equal(a, b)


def test_tma_on_concurrent_lanes_identical(oracle):
    """FHECONV_BATCH5=0 runs approach 5 one ciphertext per CUDA-stream lane: several
    k_bsgs_tma launches overlap, each with its own work-queue slot (fheconv.cu tma_rows);
    the residues equal the batched path's."""
    from paper_2306_09189_b200 import Context
    rng = np.random.default_rng(9)
    c, m, k = 16, 32, 3
    filt = rng.uniform(-1, 1, c * c * k * k)
    imgs = [rng.uniform(-1, 1, c * m * m) for _ in range(6)]
    res = {}
    for name, env in (("batched", {}), ("lanes", {"FHECONV_BATCH5": "0"})):
        old = os.environ.get("FHECONV_BATCH5")
        os.environ.pop("FHECONV_BATCH5", None)
        os.environ.update(env)
        try:
            ctx = Context.from_config("cfg3")
        finally:
            if old is None:
                os.environ.pop("FHECONV_BATCH5", None)
            else:
                os.environ["FHECONV_BATCH5"] = old
        ctx.keygen(7)
        layer = ctx.conv_layer(c, c, m, k, filt)
        ctx.gen_galois_keys(layer.steps(5))
        cts = [ctx.encrypt(ctx.encode(x), ENC_SEED + i) for i, x in enumerate(imgs)]
        outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in imgs]
        for _ in range(2):
            ctx.conv2d_batch_into(cts, layer, 5, outs)
        res[name] = [o.residues() for o in outs]
        del ctx
    for a, b in zip(res["batched"], res["lanes"]):
        assert np.array_equal(a, b)
