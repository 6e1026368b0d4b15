"""Command-line front end (reference tools/main.cpp:128-170), on ciphertexts.

    python -m paper_2306_09189_b200 run NET.json INPUT.tensor [--max-residual R] [--config cfg3]
    python -m paper_2306_09189_b200 bench NET.json INPUT.tensor [-n REPS]
    python -m paper_2306_09189_b200 decomp [LO] [HI] [--modulus S]
    python -m paper_2306_09189_b200 poly-table [--grid G]
    python -m paper_2306_09189_b200 demo [DIR]

`run` / `bench` execute the network through libfheconv on the GPU (net.py);
`decomp` and `poly-table` are host-side tables; `demo` writes a runnable
network (the reference's desk-scale two-conv layout, weights from this
package's own seeded generator) that fits cfg3's 12 levels.
Exit codes follow the reference: 2 when --max-residual is exceeded or the
bench ledgers differ between repetitions, 1 on an error.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np


def _ctx(config: str, device: int):
    from .engine import Context
    ctx = Context.from_config(config, device=device)
    ctx.keygen(7)
    return ctx


def cmd_run(a) -> int:
    from . import fixtures, net
    spec = net.load_network(a.spec)
    x = fixtures.load_tensor(a.input)
    rep = net.run_network(_ctx(a.config, a.device), spec, x)
    sys.stdout.write(rep.to_text())
    if a.max_residual > 0.0 and rep.residual_max > a.max_residual:
        print(f"FAIL: residual max {rep.residual_max:.3e} exceeds threshold {a.max_residual:.3e}")
        return 2
    return 0


def cmd_bench(a) -> int:
    from . import fixtures, net
    spec = net.load_network(a.spec)
    x = fixtures.load_tensor(a.input)
    b = net.bench_network(_ctx(a.config, a.device), spec, x, a.repetitions)
    keys = ("rotations", "hoisted_rotations", "ct_pt_mults", "ct_ct_mults", "adds", "key_switches")
    print("layer type   " + " ".join(f"{k:>17s}" for k in keys))
    for t, ops in b["per_type"].items():
        print(f"{t:<12s} " + " ".join(f"{ops.get(k, 0):17d}" for k in keys))
    print(f"deterministic across {b['repetitions']} runs: {'yes' if b['deterministic'] else 'no'}")
    return 0 if b["deterministic"] else 2


def cmd_decomp(a) -> int:
    from .engine import decompose
    print(f"{'n':>6s} {'positive':>10s} {'signed':>10s}  signed steps")
    for n in range(a.lo, min(a.hi, a.modulus - 1) + 1):
        pos, sgn = decompose(0, n, a.modulus), decompose(1, n, a.modulus)
        print(f"{n:6d} {len(pos):10d} {len(sgn):10d}  [{' '.join(str(s) for s in sgn)}]")
    return 0


def cmd_poly_table(a) -> int:
    from . import net
    relu = lambda x: x if x > 0.0 else 0.0  # noqa: E731
    print("max abs error of activation approximations on [-16, 16]")
    print(f"{'method':<18s} {'degree':>6s} {'ReLU':>10s} {'GELU':>10s}")
    xs = np.linspace(-16.0, 16.0, a.grid + 1)
    for deg in (27, 59):
        r = net.cheb_interpolate(relu, deg, 16.0)
        g = net.cheb_interpolate(net.oracle_gelu, deg, 16.0)
        er = np.abs(net.cheb_eval(r, xs) - np.maximum(xs, 0.0)).max()
        eg = np.abs(net.cheb_eval(g, xs) - np.array([net.oracle_gelu(v) for v in xs])).max()
        print(f"{'Chebyshev nodes':<18s} {deg:6d} {er:10.4f} {eg:10.4f}")
    return 0


def cmd_demo(a) -> int:
    from . import fixtures as fx
    d = a.dir
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(1234)
    unit = lambda n: rng.uniform(-1.0, 1.0, n)  # noqa: E731
    fx.save_filter(os.path.join(d, "conv1.filt"), fx.FilterTensor(4, 8, 3, 0.15 * unit(4 * 8 * 9)), 0.1 * unit(8))
    fx.save_filter(os.path.join(d, "conv2.filt"), fx.FilterTensor(8, 8, 3, 0.08 * unit(8 * 8 * 9)), 0.1 * unit(8))
    fx.save_linear(os.path.join(d, "head.lin"), fx.LinearWeights(10, 8, unit(80), unit(10)))
    fx.save_tensor(os.path.join(d, "input.tensor"), fx.ImageTensor(4, 8, unit(4 * 64)))
    spec = {"shard_size": 256, "initial_level": 12, "seed": 1, "noise": {"enabled": False},
            "bootstrap": {"auto": True},
            "layers": [{"type": "conv", "name": "conv1", "filter": "conv1.filt", "bn_scale": [1.0] * 8,
                        "bn_bias": [0.0] * 8},
                       {"type": "conv", "name": "conv2", "filter": "conv2.filt"},
                       {"type": "pool"},
                       {"type": "gelu", "degree": 27, "bound": 10.0},
                       {"type": "pool_linear", "name": "head", "weights": "head.lin"}]}
    with open(os.path.join(d, "net.json"), "w") as f:
        json.dump(spec, f, indent=2)
    print(f"demo network written to {d} (run: python -m paper_2306_09189_b200 run {d}/net.json {d}/input.tensor)")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2306_09189_b200",
                                 description="encrypted packed-tensor inference on a B200 (RNS-CKKS)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "bench"):
        p = sub.add_parser(name)
        p.add_argument("spec")
        p.add_argument("input")
        p.add_argument("--config", default="cfg3", help="CKKS parameter set (engine.CONFIGS)")
        p.add_argument("--device", type=int, default=0)
        if name == "run":
            p.add_argument("--max-residual", type=float, default=0.0)
        else:
            p.add_argument("-n", "--repetitions", type=int, default=3)
    p = sub.add_parser("decomp")
    p.add_argument("lo", type=int, nargs="?", default=0)
    p.add_argument("hi", type=int, nargs="?", default=130)
    p.add_argument("--modulus", type=int, default=4096)
    p = sub.add_parser("poly-table")
    p.add_argument("--grid", type=int, default=100000)
    p = sub.add_parser("demo")
    p.add_argument("dir", nargs="?", default="demo")
    a = ap.parse_args(argv)
    fn = {"run": cmd_run, "bench": cmd_bench, "decomp": cmd_decomp, "poly-table": cmd_poly_table,
          "demo": cmd_demo}[a.cmd]
    try:
        return fn(a)
    except Exception as e:  # the reference prints "error: ..." and exits 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
