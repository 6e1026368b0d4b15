"""Network runner on real ciphertexts (reference net.cpp:112-257):
the reference's test networks (tests/test_net.cpp, tiny_net.hpp, written as JSON
+ fixtures by its own io.cpp) run end to end through libfheconv at cfg3
(N = 2^15, 12 levels). Logits within 1e-6 of the reference's run_network, the
same per-layer level timeline, every intermediate map within 1e-6 of the
plaintext mirror, the reference's underflow error text."""
import os

import numpy as np
import pytest

from paper_2306_09189_b200 import Context, net
from test_net_host import NETDIR, NETS, load_input

pytestmark = pytest.mark.gpu
TOL = 1e-6


@pytest.fixture(scope="module")
def ctx():
    c = Context.from_config("cfg3")
    c.keygen(7)
    return c


@pytest.mark.parametrize("name", NETS)
def test_network_matches_reference(ctx, oracle, golden, name):
    spec = net.load_network(os.path.join(NETDIR, name, "net.json"))
    x = load_input(oracle, golden, name)
    ctx.ledger_reset()
    rep = net.run_network(ctx, spec, x)
    assert np.abs(rep.logits - golden[f"{name}/logits"]).max() < TOL
    assert np.abs(rep.oracle_logits - golden[f"{name}/oracle_logits"]).max() < 1e-12
    info = golden[f"{name}/info"]
    for i, l in enumerate(rep.layers):
        assert (l.level_before, l.level_after, l.depth_consumed) == tuple(int(v) for v in info[i, :3]), (name, i)
        assert l.max_abs_err < TOL, (name, l.name, l.max_abs_err)
    assert rep.residual_max < TOL
    assert rep.totals["ct_ct_mults"] > 0 or all(l.type != "gelu" for l in rep.layers)
    assert "residual mean" in rep.to_text()


def test_tiny_network_gelu_consumes_series_depth(ctx, oracle, golden):
    """test_net.cpp:27-35: the folded bound keeps the activation prescaled (bits(27) = 5 levels)."""
    spec = net.load_network(os.path.join(NETDIR, "net_tiny", "net.json"))
    rep = net.run_network(ctx, spec, load_input(oracle, golden, "net_tiny"), check_layers=False)
    g = rep.layers[3]
    assert g.type == "gelu" and g.level_before - g.level_after == 5


def test_level_underflow_is_a_structured_error(ctx, oracle, golden):
    """test_net.cpp:62-73: without bootstraps, initial level 6 underflows at the activation."""
    spec = net.load_network(os.path.join(NETDIR, "net_tiny", "net.json"))
    spec.initial_level = 6
    with pytest.raises(RuntimeError) as e:
        net.run_network(ctx, spec, load_input(oracle, golden, "net_tiny"))
    assert str(e.value) == bytes(golden["net_tiny/underflow_l6"]).decode()


def test_bench_network_ledgers_deterministic(ctx, oracle, golden):
    """bench_network (net.cpp:285-310): ledgers identical across repetitions."""
    spec = net.load_network(os.path.join(NETDIR, "net_tiny", "net.json"))
    b = net.bench_network(ctx, spec, load_input(oracle, golden, "net_tiny"), 2)
    assert b["deterministic"] and b["per_type"]["conv"]["ct_pt_mults"] > 0


@pytest.mark.parametrize("c,m", [(4, 32), (8, 32), (16, 32), (2, 16)])
def test_pooled_output_feeds_the_next_convolution(oracle, c, m):
    """test_pool.cpp:224-252: a pooled map (rep 4 / 2 / 1, permuted tau, duplication) feeds
    fhe_conv_layer_create_packed; decrypted and unpacked it equals conv(avgpool(x)) (cfg1)."""
    from paper_2306_09189_b200 import fixtures as fx
    from test_gpu_parity import pair
    p = pair(oracle, "cfg1")
    s = p.ctx.slots
    img, filt = oracle.make_inputs(c, m, 3, c, 500 + c, 600 + c, 0)
    x = fx.ImageTensor(c, m, img)
    slots, d, mode = net.pack_slots(x, s)
    keys = net._Keys(p.ctx)
    cts = [p.ctx.encrypt(p.ctx.encode(v), 9100 + u) for u, v in enumerate(slots)]
    pk = net.PackedCiphertexts(cts, m, c, np.arange(c), 1, d, mode)
    pooled = net._downsample(p.ctx, keys, pk, True, 1.0)
    k = fx.FilterTensor(c, c, 3, filt)
    out = net._conv(p.ctx, keys, pooled, k, np.zeros(0), 1.0)
    got = net.unpack_slots(out, [p.ctx.decrypt(o) for o in out.shards], s)
    want = net.oracle_conv(net.oracle_avgpool2x2(x), k).data
    assert np.abs(got - want).max() < TOL


def test_cli_run_and_bench_demo(tmp_path, capsys):
    """`run` / `bench` of the demo network on the GPU (tools/main.cpp:23-42 semantics)."""
    from paper_2306_09189_b200.__main__ import main
    d = str(tmp_path / "demo")
    assert main(["demo", d]) == 0
    assert main(["run", f"{d}/net.json", f"{d}/input.tensor", "--max-residual", "1e-6"]) == 0
    out = capsys.readouterr().out
    assert "residual mean" in out and "gelu" in out
    assert main(["bench", f"{d}/net.json", f"{d}/input.tensor", "-n", "2"]) == 0
    assert "deterministic across 2 runs: yes" in capsys.readouterr().out
