"""Randomised geometry sweep at cfg1 (N=2^13): single-shard, multi-shard and channel-shard convs,
every schedule on the single-shard layers, batched and single; decrypted vs a float64 conv."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402


def ref_conv(img, filt, c, co, m, k):
    x = img.reshape(c, m, m)
    w = filt.reshape(c, co, k, k)
    h = k // 2
    xp = np.pad(x, ((0, 0), (h, h), (h, h)))
    return sum(np.einsum("fg,fij->gij", w[:, :, r, t], xp[:, r:r + m, t:t + m]) for r in range(k) for t in range(k))


ctx = Context.from_config("cfg1")
ctx.keygen(7)
s = ctx.slots
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
fails = 0
cases = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    m = int(rng.choice([4, 8, 16, 32, 64, 128]))
    k = int(rng.choice([1, 3, 5, 7]))
    if k // 2 >= m:
        continue
    c = int(rng.choice([1, 2, 4, 8, 16]))
    co = int(rng.choice([1, 2, 4, 8, 16]))
    if c * m * m > 16 * s or co * m * m > 16 * s:
        continue
    img = rng.uniform(-1, 1, c * m * m)
    filt = rng.uniform(-1, 1, c * co * k * k) * 0.5
    ref = ref_conv(img, filt, c, co, m, k)
    try:
        if m * m <= s and c * m * m < s and co * m * m > s:  # duplicated input, several output shards
            d = s // (c * m * m)
            layer = ctx.conv_layer_packed(c, co, m, k, filt, t=1, d=d)
            ctx.gen_galois_keys(layer.steps())
            ct = ctx.encrypt(ctx.encode(np.tile(img, d)), 9000 + it)
            outs = ctx.conv2d_shards([ct], layer)
            z = s // (m * m)
            ys = [ctx.decrypt(o) for o in outs]
            got = np.stack([ys[g // z][(g % z) * m * m:(g % z + 1) * m * m] for g in range(co)])
            err = np.abs(got.ravel() - ref.ravel()).max()
            tag = f"dup d={d} -> {len(outs)} shards"
        elif m * m <= s and c * m * m <= s and co * m * m <= s:  # single shard (duplicated when small)
            d = s // (c * m * m)
            layer = ctx.conv_layer_packed(c, co, m, k, filt, t=1, d=d) if d > 1 else ctx.conv_layer(c, co, m, k, filt)
            if d > 1:
                ctx.gen_galois_keys(layer.steps())
                ct = ctx.encrypt(ctx.encode(np.tile(img, d)), 9000 + it)
                outs = ctx.conv2d_shards([ct], layer)
                got = outs[0]
                z = s // (m * m)
                y = ctx.decrypt(got)
                got_img = np.stack([y[((g) % z) * m * m:((g) % z + 1) * m * m] for g in range(co)])
                err = np.abs(got_img.ravel() - ref.ravel()).max()
                tag = f"dup d={d}"
            else:
                ctx.gen_galois_keys(layer.steps(0))
                ct = ctx.encrypt(ctx.encode(img), 9000 + it)
                errs = []
                for ap in (0, 1, 2, 3, 5):
                    o = ctx.conv2d(ct, layer, ap)
                    errs.append(np.abs(ctx.decrypt(o)[: co * m * m] - ref.ravel()).max())
                    ob = ctx.conv2d_batch([ct, ct], layer, ap)[1]
                    errs.append(np.abs(ctx.decrypt(ob)[: co * m * m] - ref.ravel()).max())
                err = max(errs)
                tag = "single all-approaches"
        else:
            layer = ctx.conv_layer_shards(c, co, m, k, filt)
            ctx.gen_galois_keys(layer.steps())
            if m * m > s:
                chunks = list(img.reshape(-1, s))
            else:
                chunks = list(img.reshape(-1, s))
            cts = [ctx.encrypt(ctx.encode(x), 9000 + u) for u, x in enumerate(chunks)]
            outs = ctx.conv2d_shards(cts, layer)
            if m * m > s:
                got = np.concatenate([ctx.decrypt(o) for o in outs])
                err = np.abs(got - ref.ravel()).max()
                tag = "channel shards"
            else:
                z = s // (m * m)
                ys = [ctx.decrypt(o) for o in outs]
                got = np.stack([ys[g // z][(g % z) * m * m:(g % z + 1) * m * m] for g in range(co)]) if co >= z else \
                    np.stack([ys[0][(g % z) * m * m:(g % z + 1) * m * m] for g in range(co)])
                err = np.abs(got.ravel() - ref.ravel()).max()
                tag = "image shards"
        cases += 1
        ok = err < 1e-6
        fails += not ok
        print(f"{'ok  ' if ok else 'FAIL'} c={c} co={co} m={m} k={k} {tag}: {err:.2e}", flush=True)
    except Exception as e:
        print(f"ERR  c={c} co={co} m={m} k={k}: {type(e).__name__}: {e}", flush=True)
print(f"{cases} cases, {fails} failures")
