import sys, time, numpy as np, gc
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
ctx = Context.from_config("cfg3"); ctx.keygen(7)
M = 32
stencil = [kk * M + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(stencil)
ct = ctx.encrypt(ctx.encode(np.random.default_rng(0).uniform(-1, 1, 16384)), 1)
for rep in range(3):
    ctx.synchronize()
    ts = []
    for _ in range(20):
        t = time.perf_counter(); hs = ctx.rotate_hoisted(ct, stencil); ts.append(time.perf_counter() - t)
    ctx.synchronize()
    print("host ms per call: max %.2f median %.3f" % (1e3 * max(ts), 1e3 * sorted(ts)[10]), [round(1e3*x, 2) for x in ts[:20]], flush=True)
