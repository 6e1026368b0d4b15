import sys, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
ctx = Context.from_config("cfg3"); ctx.keygen(7)
M = 32
stencil = [kk * M + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(stencil)
ct = ctx.encrypt(ctx.encode(np.random.default_rng(0).uniform(-1, 1, 16384)), 1)
for _ in range(3): hs = ctx.rotate_hoisted(ct, stencil)
ctx.synchronize(); ctx.timer_start()
for _ in range(20): hs = ctx.rotate_hoisted(ct, stencil)
ms = ctx.timer_stop()
print("hoisted rot/s", 20 * len(stencil) / (ms / 1e3))
for B in (4, 16):
    cts = [ctx.encrypt(ctx.encode(np.random.default_rng(i).uniform(-1, 1, 16384)), 10 + i) for i in range(B)]
    for _ in range(2): hs = ctx.rotate_hoisted_batch(cts, stencil)
    ctx.synchronize(); ctx.timer_start()
    for _ in range(5): hs = ctx.rotate_hoisted_batch(cts, stencil)
    ms = ctx.timer_stop()
    print(f"batched B={B} hoisted rot/s", 5 * B * len(stencil) / (ms / 1e3))
