"""Network runner host side, CPU only: fixture I/O in the
reference's formats (io.cpp:31-103), JSON loading (net.cpp:51-110) and the
plaintext mirror (net.cpp:166-223) against the reference's own files and
outputs (tests/golden/net/*, written by the reference's savers; golden logits
from its run_network, tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from paper_2306_09189_b200 import fixtures as fx
from paper_2306_09189_b200 import net

NETDIR = os.path.join(os.path.dirname(__file__), "golden", "net")
NETS = ["net_tiny", "net_stride2", "net_gelu_first", "net_channel"]


def load_input(oracle, golden, name):
    p = os.path.join(NETDIR, name, "input.tensor")
    if os.path.exists(p):
        x = fx.load_tensor(p)
    else:  # net_channel: random_tensor(mt19937_64(77), 2, 256) (ref_shim build_net)
        img, _ = oracle.make_inputs(2, 256, 1, 1, 77, 0, 0)
        x = fx.ImageTensor(2, 256, img)
    assert np.array_equal(np.array([x.data.sum(), np.abs(x.data).sum()]), golden[f"{name}/input_sum"])
    return x


@pytest.mark.parametrize("name", NETS)
def test_fixtures_round_trip_byte_identical(tmp_path, name):
    """our savers reproduce the reference's fixture files byte for byte."""
    d = os.path.join(NETDIR, name)
    for f in sorted(os.listdir(d)):
        src = os.path.join(d, f)
        dst = str(tmp_path / f)
        if f.endswith(".filt"):
            k, b = fx.load_filter(src)
            fx.save_filter(dst, k, b)
        elif f.endswith(".lin"):
            fx.save_linear(dst, fx.load_linear(src))
        elif f.endswith(".tensor"):
            fx.save_tensor(dst, fx.load_tensor(src))
        else:
            continue
        assert open(src).read() == open(dst).read(), f


def test_fixture_errors(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        fx.load_tensor(str(tmp_path / "missing.tensor"))
    p = tmp_path / "t.tensor"
    p.write_text("2 4\n1 2 3\n")
    with pytest.raises(RuntimeError, match="truncated fixture"):
        fx.load_tensor(str(p))
    p.write_text("x")
    with pytest.raises(RuntimeError, match="bad tensor header"):
        fx.load_tensor(str(p))
    poly = net.cheb_interpolate(net.oracle_gelu, 27, 10.0)
    fx.save_poly(str(tmp_path / "p.poly"), poly)
    p2 = fx.load_poly(str(tmp_path / "p.poly"))
    assert p2.bound == poly.bound and np.array_equal(p2.coeffs, poly.coeffs)


def test_cheb_interpolate_matches_reference(golden):
    """act.cpp:103-125 restated: the GELU interpolant equals the reference's coefficients."""
    co = golden["cheb_cfg3_gelu27_pre/coeffs"]
    ours = net.cheb_interpolate(net.oracle_gelu, 27, 10.0).coeffs
    assert np.abs(ours - co).max() < 1e-15


@pytest.mark.parametrize("name", NETS)
def test_mirror_matches_reference_oracle_logits(oracle, golden, name):
    """load_network + the plaintext mirror give the reference's oracle logits."""
    spec = net.load_network(os.path.join(NETDIR, name, "net.json"))
    x = load_input(oracle, golden, name)
    _, logits = net.mirror_network(spec, x)
    assert np.abs(logits - golden[f"{name}/oracle_logits"]).max() < 1e-12


def test_required_levels_match_reference(golden):
    """per-layer level consumption of the golden runs (12 levels, no bootstraps)."""
    for name in NETS:
        spec = net.load_network(os.path.join(NETDIR, name, "net.json"))
        _, pre, _ = net._plan(spec)
        depth = golden[f"{name}/info"][:, 2]
        for i, ly in enumerate(spec.layers):
            assert net.required_level(ly, pre[i]) == depth[i], (name, i)


def test_malformed_networks_rejected(tmp_path):
    p = tmp_path / "n.json"
    p.write_text('{"layers": [{"type": "dropout"}]}')
    with pytest.raises(RuntimeError, match="unknown layer type: dropout"):
        net.load_network(str(p))
    with pytest.raises(RuntimeError, match="cannot open"):
        net.load_network(str(tmp_path / "none.json"))


def test_slot_feature_map_and_unpack():
    """pack.cpp:84-129 restated over packings with duplication, rep and tau."""
    s = 64
    x = fx.ImageTensor(2, 4, np.arange(32.0))
    slots, d, mode = net.pack_slots(x, s)
    assert (d, mode, len(slots)) == (2, 0, 1)
    p = net.PackedCiphertexts([None], 4, 2, np.arange(2), 1, d, mode)
    assert np.array_equal(net.unpack_slots(p, slots, s), x.data)
    fm = net.slot_feature_map(p, s)
    assert (fm[0, 32:] == -1).all() and np.array_equal(fm[0, :32], np.arange(32))
    # rep 2, tau (1, 0): block g holds channel tau[(g // 2) % 2]
    p2 = net.PackedCiphertexts([None], 2, 2, np.array([1, 0]), 2, 4, 0)
    fm2 = net.slot_feature_map(p2, 32)
    assert np.array_equal(fm2[0, :4], 4 + np.arange(4)) and (fm2[0, 4:8] == -1).all()
    assert np.array_equal(fm2[0, 8:12], np.arange(4))


def test_cli_decomp_matches_reference_tables(golden, capsys):
    """`decomp` (tools/main.cpp:62-72): positive / signed lengths equal the reference's."""
    from paper_2306_09189_b200.__main__ import main
    assert main(["decomp", "0", "200", "--modulus", "4096"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()[1:]
    lens = golden["decomp4096/lens"]
    for ln in lines:
        n, pos, sgn = (int(x) for x in ln.split()[:3])
        assert (pos, sgn) == (int(lens[0][n]), int(lens[1][n])), n


def test_cli_demo_and_poly_table(tmp_path, capsys):
    from paper_2306_09189_b200.__main__ import main
    d = str(tmp_path / "demo")
    assert main(["demo", d]) == 0
    spec = net.load_network(os.path.join(d, "net.json"))
    assert [l.type for l in spec.layers] == ["conv", "conv", "pool", "gelu", "pool_linear"]
    _, pre, _ = net._plan(spec)
    assert sum(net.required_level(l, pre[i]) for i, l in enumerate(spec.layers)) <= 12  # fits cfg3
    assert main(["poly-table", "--grid", "2000"]) == 0
    out = capsys.readouterr().out
    assert "Chebyshev nodes" in out
    assert main(["run", os.path.join(d, "missing.json"), os.path.join(d, "input.tensor")]) == 1
