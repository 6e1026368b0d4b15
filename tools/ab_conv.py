"""A/B timing of one libfheconv build (FHECONV_LIB=...): cfg3 batched conv, prints ms/conv and an output hash."""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
AP = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg3"
geo = {"cfg1": (4, 32, 3), "cfg3": (16, 32, 3), "cfg4": (8, 64, 5)}[cfg]
ctx = Context.from_config(cfg)
ctx.keygen(7)
c, m, k = geo
rng = np.random.default_rng(0)
layer = ctx.conv_layer(c, c, m, k, rng.uniform(-1, 1, c * c * k * k))
ctx.gen_galois_keys(layer.steps(AP))
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c * m * m)), 9000 + i) for i in range(B)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in range(B)]
for _ in range(3):
    ctx.conv2d_batch_into(cts, layer, AP, outs)
ctx.synchronize()
best = 1e9
for rep in range(5):
    ctx.timer_start()
    for _ in range(4):
        ctx.conv2d_batch_into(cts, layer, AP, outs)
    best = min(best, ctx.timer_stop() / 4 / B)
h = hashlib.sha1(b"".join(o.residues().tobytes() for o in outs)).hexdigest()[:16]
print(f"{cfg} ap={AP} B={B}: {best:.4f} ms/conv ({1e3 / best:.0f} conv/s) hash {h}")
