"""The single-launch cluster NTT (k_ntt_fused: one thread-block cluster per residue row, the
column -> row intermediate exchanged through distributed shared memory; FHE_NTT_FUSED=1)
gives the same residues as the default two-launch transform, at every ring size with a
cluster form (N = 2^13 cfg1, 2^14 cfg2, 2^15 cfg3): encryption (forward NTT), a conv
(ModUp forward transforms, inverse transforms, the fused ModDown + rescale epilogue) and
hoisted rotations (ModDown epilogue through output pointer tables).

The transform itself is pinned to the golden model by tests/test_gpu_parity.py (default
path); this test pins the opt-in kernel to the default one."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _run(cfg, geo):
    from paper_2306_09189_b200 import Context
    rng = np.random.default_rng(11)
    ctx = Context.from_config(cfg)
    ctx.keygen(7)
    out = []
    n_slots = ctx.slots
    ct = ctx.encrypt(ctx.encode(rng.uniform(-1, 1, n_slots)), 9001)
    out.append(ct.residues().copy())
    steps = [1, -1, 32, -33]
    ctx.gen_galois_keys(steps)
    for r in ctx.rotate_hoisted(ct, steps):
        out.append(r.residues().copy())
    if geo is not None:
        c, m, k = geo
        filt = rng.uniform(-1, 1, c * c * k * k)
        layer = ctx.conv_layer(c, c, m, k, filt)
        for ap in (5, 2):
            ctx.gen_galois_keys(layer.steps(ap))
            cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c * m * m)), 9100 + i) for i in range(3)]
            for o in ctx.conv2d_batch(cts, layer, ap):
                out.append(o.residues().copy())
    return out


@pytest.mark.parametrize("cfg,geo", [("cfg1", (4, 32, 3)), ("cfg2", None), ("cfg3", (16, 32, 3))])
def test_cluster_ntt_matches_two_launch_transform(cfg, geo):
    old = os.environ.get("FHE_NTT_FUSED")
    try:
        os.environ.pop("FHE_NTT_FUSED", None)
        ref = _run(cfg, geo)
        os.environ["FHE_NTT_FUSED"] = "1"
        got = _run(cfg, geo)
    finally:
        if old is None:
            os.environ.pop("FHE_NTT_FUSED", None)
        else:
            os.environ["FHE_NTT_FUSED"] = old
    assert len(ref) == len(got)
    for i, (a, b) in enumerate(zip(ref, got)):
        assert np.array_equal(a, b), f"{cfg}: output {i} differs between the cluster and two-launch NTT"
