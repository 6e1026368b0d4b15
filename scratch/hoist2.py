import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
ctx = Context.from_config("cfg3"); ctx.keygen(7)
M = 32
stencil = [kk * M + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(stencil)
ct = ctx.encrypt(ctx.encode(np.random.default_rng(0).uniform(-1, 1, 16384)), 1)
for rep in range(3):
    ctx.synchronize(); t = time.perf_counter(); ctx.timer_start()
    for _ in range(20): hs = ctx.rotate_hoisted(ct, stencil)
    ms = ctx.timer_stop(); w = time.perf_counter() - t
    print(f"single: {20*8/(ms/1e3):.0f} rot/s device, {20*8/w:.0f} wall", flush=True)
ctx.prof_reset(); ctx.prof_enable(True)
for _ in range(5): hs = ctx.rotate_hoisted(ct, stencil)
ctx.prof_enable(False)
for cl in ["ntt", "ntt_modup", "ntt_moddown", "ks_multi", "moddown"]:
    print(cl, ctx.prof_get_bytes(cl))
for B in (4, 16):
    cts = [ctx.encrypt(ctx.encode(np.random.default_rng(i).uniform(-1, 1, 16384)), 10 + i) for i in range(B)]
    for rep in range(3):
        ctx.synchronize(); t = time.perf_counter(); ctx.timer_start()
        for _ in range(5): hs = ctx.rotate_hoisted_batch(cts, stencil)
        ms = ctx.timer_stop(); w = time.perf_counter() - t
        print(f"batched B={B}: {5*B*8/(ms/1e3):.0f} rot/s device, {5*B*8/w:.0f} wall", flush=True)
