"""The opt-in NTT kernels give the same residues as the default two-launch transform:

* the single-launch cluster NTT (k_ntt_fused: one thread-block cluster per residue row, the
  column -> row intermediate exchanged through distributed shared memory; FHE_NTT_FUSED=1),
  at every ring size with a cluster form (N = 2^13 cfg1, 2^14 cfg2, 2^15 cfg3);
* the row phase with shared-memory twiddles reused over R rows (k_ntt_rows_tw; FHE_NTT_TWR=R);
* the forward row phase that prefetches the next row's residues (k_ntt_rows_pf; FHE_NTT_PF=R).

Covered: encryption (forward NTT), batched convs (ModUp forward transforms, inverse
transforms, the fused ModDown + rescale epilogue) and hoisted rotations (ModDown epilogue
through output pointer tables). All three were measured slower than the default on the
B200 (profiles/ab_r02_ntt_cluster.txt, profiles/ab_r02_ntt_twiddles.txt,
profiles/ab_r02_ntt_prefetch.txt) and stay opt-in.

The transform itself is pinned to the golden model by tests/test_gpu_parity.py (default
path); this test pins the opt-in kernel to the default one."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _run(cfg, geo, nct=3):
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
            cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c * m * m)), 9100 + i) for i in range(nct)]
            for o in ctx.conv2d_batch(cts, layer, ap):
                out.append(o.residues().copy())
    return out


def _ab(var, value, cfg, geo, nct):
    old = os.environ.get(var)
    try:
        os.environ.pop(var, None)
        ref = _run(cfg, geo, nct)
        os.environ[var] = value
        got = _run(cfg, geo, nct)
    finally:
        if old is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = old
    assert len(ref) == len(got)
    for i, (a, b) in enumerate(zip(ref, got)):
        assert np.array_equal(a, b), f"{cfg}: output {i} differs between {var}={value} and the default NTT"


@pytest.mark.parametrize("cfg,geo", [("cfg1", (4, 32, 3)), ("cfg2", None), ("cfg3", (16, 32, 3))])
def test_cluster_ntt_matches_two_launch_transform(cfg, geo):
    _ab("FHE_NTT_FUSED", "1", cfg, geo, 3)


@pytest.mark.parametrize("cfg,geo,nct,r", [("cfg1", (4, 32, 3), 16, "4"), ("cfg3", (16, 32, 3), 16, "8")])
def test_shared_twiddle_row_phase_matches_default(cfg, geo, nct, r):
    # batches of 16: enough rows per prime for the R-row groups to be used (two waves of CTAs)
    _ab("FHE_NTT_TWR", r, cfg, geo, nct)


def test_prefetching_row_phase_matches_default():
    _ab("FHE_NTT_PF", "4", "cfg3", (16, 32, 3), 16)
