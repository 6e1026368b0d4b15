"""TMA staging edge cases (run with FHECONV_GRAPHS=0 under a short timeout): kernels 3/5/7 (plaintext
boxes across giant chunks, cfg1) and batches of 1, 2, 3, 5 and 6 ciphertexts (partial source groups)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import CONFIGS, Context  # noqa: E402
ctx = Context(**CONFIGS["cfg1"])
ctx.keygen(7)
rng = np.random.default_rng(3)
img = rng.uniform(-1, 1, 4096)
for k in (3, 5, 7):
    filt = rng.uniform(-1, 1, 16 * k * k)
    layer = ctx.conv_layer(4, 4, 32, k, filt)
    ctx.gen_galois_keys(layer.steps(0))
    for B in (1, 2, 3, 5, 6):
        cts = [ctx.encrypt(ctx.encode(img), 9000 + i) for i in range(B)]
        outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level - 1), 1) for _ in range(B)]
        ctx.conv2d_batch_into(cts, layer, 0, outs)
        ctx.synchronize()
        print("k", k, "B", B, "ok", flush=True)
