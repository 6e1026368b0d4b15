import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
ctx = Context.from_config("cfg3"); ctx.keygen(7)
M = 32
stencil = [kk * M + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(stencil)
for B in (1, 4, 8, 16):
    cts = [ctx.encrypt(ctx.encode(np.random.default_rng(i).uniform(-1, 1, 16384)), 10 + i) for i in range(B)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8)), 1) for _ in range(B * 8)]
    for _ in range(3): ctx.rotate_hoisted_batch_into(cts, stencil, outs)
    for rep in range(3):
        ctx.synchronize(); ctx.timer_start()
        for _ in range(10): ctx.rotate_hoisted_batch_into(cts, stencil, outs)
        ms = ctx.timer_stop()
        print(f"batched_into B={B}: {10*B*8/(ms/1e3):.0f} rot/s", flush=True)
