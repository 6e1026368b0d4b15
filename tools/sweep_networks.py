"""Randomised network sweep at cfg3 (12 levels): conv (+stride 2) / pool / gelu / linear or
pool_linear stacks over random geometries through net.run_network; every layer's decrypted map
and the logits checked against the plaintext mirror."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context, fixtures as fx, net  # noqa: E402

ctx = Context.from_config("cfg3")
ctx.keygen(7)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_ok = n_bad = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    c = int(rng.choice([1, 2, 4, 8, 16]))
    m = int(rng.choice([8, 16, 32, 64, 128, 256]))
    if c * m * m > 8 * 16384:
        continue
    layers, levels, cc, mm = [], 0, c, m
    while True:
        kind = rng.choice(["conv", "conv2", "pool"]) if mm >= 4 else "conv"
        if kind == "pool" and levels + 3 + 7 <= 12 and mm >= 4:
            layers.append(net.LayerSpec(type="pool", name=f"pool{len(layers)}"))
            levels += 3
            mm //= 2
        elif kind in ("conv", "conv2"):
            stride = 2 if kind == "conv2" and mm >= 4 else 1
            need = 3 if stride == 2 else 1
            if levels + need + 7 > 12:
                break
            co = int(rng.choice([1, 2, 4, 8]))
            k = int(rng.choice([1, 3, 5]))
            if k // 2 >= mm:
                k = 1
            w = rng.uniform(-1, 1, cc * co * k * k) * (0.6 / (cc * k))
            layers.append(net.LayerSpec(type="conv", name=f"conv{len(layers)}", filter=fx.FilterTensor(cc, co, k, w),
                                        bias=rng.uniform(-0.1, 0.1, co), stride=stride))
            levels += need
            cc = co
            if stride == 2:
                mm //= 2
        if rng.random() < 0.35 or levels >= 5:
            break
    layers.append(net.LayerSpec(type="gelu", name="gelu", degree=int(rng.choice([7, 15, 27])), bound=4.0))
    no = int(rng.integers(1, 6))
    if rng.random() < 0.5:
        layers.append(net.LayerSpec(type="pool_linear", name="head",
                                    weights=fx.LinearWeights(no, cc, rng.uniform(-1, 1, no * cc), rng.uniform(-1, 1, no))))
    else:
        nin = cc * mm * mm
        layers.append(net.LayerSpec(type="linear", name="fc",
                                    weights=fx.LinearWeights(no, nin, rng.uniform(-1, 1, no * nin) / np.sqrt(nin),
                                                             rng.uniform(-1, 1, no))))
    spec = net.NetworkSpec(shard_size=16384, initial_level=12, layers=layers)
    x = fx.ImageTensor(c, m, rng.uniform(-1, 1, c * m * m))
    desc = f"{c}x{m}x{m}: " + " ".join(
        (f"conv{l.filter.c_out}k{l.filter.kappa}s{l.stride}" if l.type == "conv" else l.type) for l in layers)
    try:
        rep = net.run_network(ctx, spec, x)
        worst = max(l.max_abs_err for l in rep.layers)
        ok = worst < 1e-6 and rep.residual_max < 1e-6
        n_ok += ok
        n_bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {desc}  worst layer err {worst:.2e} levels "
              f"{[(l.level_before, l.level_after) for l in rep.layers]}", flush=True)
    except Exception as e:
        n_bad += 1
        print(f"ERR  {desc}: {type(e).__name__}: {e}", flush=True)
print(f"{n_ok} ok, {n_bad} failed")
