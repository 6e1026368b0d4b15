"""Operation-count laws of the reference (test_conv.cpp:244-276,
acceptance.cpp:205-243) hold for the CKKS path's ledger, plus error
behaviour matching the reference's exception messages."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2306_09189_b200 import Context
    c = Context.from_config("cfg1")
    c.keygen(7)
    return c


def run(ctx, oracle, approach, name="cfg1"):
    img, filt = oracle.make_inputs(4, 32, 3, 4, 1000, 2000, 0)
    layer = ctx.conv_layer(4, 4, 32, 3, filt)
    ctx.gen_galois_keys(layer.steps())
    ct = ctx.encrypt(ctx.encode(img), 9000)
    ctx.ledger_reset()
    out = ctx.conv2d(ct, layer, approach)
    return ctx.ledger(), out, ct


@pytest.mark.parametrize("approach,plan", [(1, 1), (2, 2)])
def test_ledger_matches_reference(ctx, oracle, golden, approach, plan):
    lg, out, ct = run(ctx, oracle, approach)
    ref = [int(x) for x in golden[f"cfg1/ledger{plan}"]]
    got = [lg[f] for f in ("rotations", "hoisted_rotations", "hoist_groups", "ct_pt_mults", "ct_ct_mults", "adds",
                           "bootstraps", "max_depth_consumed", "distinct_amounts")]
    assert got == ref
    assert out.level == ct.level - 1  # one level per conv (test_conv.cpp:210-223)


def test_ckks_work_counts(ctx, oracle):
    lg, _, _ = run(ctx, oracle, 2)
    # Approach 2: one ModUp of src + one per channel-rotated copy; c-1 + c(k^2-1) key switches;
    # one ModDown per channel rotation (2 polys) + one fused ModDown pair; one rescale
    assert lg["modups"] == 1 + 4
    assert lg["key_switches"] == 3 + 4 * 8
    assert lg["moddowns"] == 2 * 3 + 2
    assert lg["rescales"] == 1
    lg, _, _ = run(ctx, oracle, 1)
    assert lg["modups"] == 1 + 9
    assert lg["key_switches"] == 8 + 9 * 3
    # fused BSGS (approach 5): c kappa - 1 = 11 hoisted baby key switches from one
    # ModUp, kappa - 1 = 2 giant steps (ModDown + ModUp + key switch each)
    lg, _, _ = run(ctx, oracle, 5)
    assert lg["modups"] == 1 + 2
    assert lg["key_switches"] == 11 + 2
    assert lg["hoist_groups"] == 1 and lg["hoisted_rotations"] == 12 and lg["rotations"] == 2
    assert lg["rescales"] == 1


def test_error_messages(ctx):
    from paper_2306_09189_b200 import FheError, InvalidArgument
    z = np.zeros(ctx.slots)
    ct = ctx.encrypt(ctx.encode(z), 1)
    with pytest.raises(InvalidArgument, match="empty rotation batch"):
        ctx.rotate_hoisted(ct, [])
    with pytest.raises(InvalidArgument, match="slot count must be a power of two"):
        ctx.encode(np.zeros(3))
    low = ctx.encrypt(ctx.encode(z, level=0), 1)
    with pytest.raises(FheError, match="depth exhausted"):
        ctx.rescale(low)
    with pytest.raises(InvalidArgument, match="insufficient capacity"):
        ctx.conv_layer(4, 8, 32, 3, np.zeros(4 * 8 * 9))
    with pytest.raises(InvalidArgument, match="kernel size must be odd"):
        ctx.conv_layer(4, 4, 32, 2, np.zeros(4 * 4 * 4))
    with pytest.raises(FheError, match="missing Galois key"):
        ctx.rotate(ct, 12345)


def test_zero_filter_and_identity(ctx, oracle):
    """all-empty plaintexts (Acc::finish zero product, conv.cpp:25-28) and the identity filter."""
    img, _ = oracle.make_inputs(4, 32, 3, 4, 1000, 2000, 0)
    ct = ctx.encrypt(ctx.encode(img), 9000)
    zero = ctx.conv_layer(4, 4, 32, 3, np.zeros(4 * 4 * 9))
    assert np.abs(ctx.decrypt(ctx.conv2d(ct, zero, 2))).max() < 1e-6
    ident = np.zeros((4, 4, 3, 3))
    for f in range(4):
        ident[f, f, 1, 1] = 1.0
    layer = ctx.conv_layer(4, 4, 32, 3, ident.ravel())
    for ap in (1, 2, 3, 4, 5):
        assert np.abs(ctx.decrypt(ctx.conv2d(ct, layer, ap)) - img).max() < 1e-6
    for ap in (3, 4, 5):
        assert np.abs(ctx.decrypt(ctx.conv2d(ct, zero, ap))).max() < 1e-6


def test_cxx_engine_demo_runs():
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = "/tmp/fheconv_engine_demo_gpu"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cxx", "engine_demo.cpp"), "-o", exe,
                    "-L", os.path.join(root, "paper_2306_09189_b200"), "-lfheconv",
                    f"-Wl,-rpath,{os.path.join(root, 'paper_2306_09189_b200')}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_graph_replay_keeps_ledger_and_results(ctx, oracle):
    """batched convs are captured into a CUDA graph once and replayed; the replay re-applies
    the capture's ledger counters and produces the same residues."""
    img, filt = oracle.make_inputs(4, 32, 3, 4, 1000, 2000, 0)
    layer = ctx.conv_layer(4, 4, 32, 3, filt)
    ctx.gen_galois_keys(layer.steps())
    cts = [ctx.encrypt(ctx.encode(np.roll(img, i)), 9000 + i) for i in range(3)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in range(3)]
    deltas, results = [], []
    for _ in range(3):  # capture, replay, replay
        ctx.ledger_reset()
        ctx.conv2d_batch_into(cts, layer, 5, outs)
        lg = ctx.ledger()
        deltas.append({k: lg[k] for k in ("rotations", "hoisted_rotations", "ct_pt_mults", "key_switches", "modups",
                                          "moddowns", "rescales", "kernel_launches")})
        results.append([o.residues() for o in outs])
    launches = [d.pop("kernel_launches") for d in deltas]
    assert deltas[0] == deltas[1] == deltas[2] and deltas[0]["key_switches"] > 0
    # the first call also encodes the layer's rotated plaintexts (one-time setup)
    assert launches[1] == launches[2] > 0 and launches[0] >= launches[1]
    for r in results[1:]:
        for a, b in zip(results[0], r):
            assert np.array_equal(a, b)


def test_graph_cache_never_replays_a_freed_layer(oracle):
    """CUDA graphs are keyed by a per-layer id, not the host address: creating and freeing
    layers of different geometry over the same ciphertext buffers always gives the new
    layer's result (a stale graph would replay the freed layer's kernels)."""
    import gc
    import numpy as np
    from paper_2306_09189_b200 import CONFIGS, Context
    ctx = Context(**CONFIGS["cfg1"])
    ctx.keygen(7)
    rng = np.random.default_rng(3)
    img = rng.uniform(-1, 1, 4096)
    ct = ctx.encrypt(ctx.encode(img), 9000)
    out = ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1)
    for k in (3, 5, 3, 7):
        filt = rng.uniform(-1, 1, 16 * k * k)
        layer = ctx.conv_layer(4, 4, 32, k, filt)
        ctx.gen_galois_keys(layer.steps(0))
        for _ in range(2):
            ctx.conv2d_into(ct, layer, 0, out)
        x = img.reshape(4, 32, 32)
        w = filt.reshape(4, 4, k, k)
        h = k // 2
        xp = np.pad(x, ((0, 0), (h, h), (h, h)))
        ref = sum(np.einsum("fg,fij->gij", w[:, :, r, s], xp[:, r:r + 32, s:s + 32])
                  for r in range(k) for s in range(k))
        assert np.abs(ctx.decrypt(out) - ref.ravel()).max() < 1e-6
        del layer
        gc.collect()
