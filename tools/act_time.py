import time, numpy as np, torch, math, sys
sys.path.insert(0, "oracle")
from paper_2306_09189_b200 import Context
import pyoracle as po
ctx = Context.from_config("cfg3"); ctx.keygen(7); ctx.gen_relin_key()
x = np.random.default_rng(1).uniform(-16, 16, ctx.slots)
gelu = lambda v: v * 0.5 * (1 + math.erf(v / math.sqrt(2)))
for deg, pre in ((59, False), (27, True)):
    co = po.cheb_interpolate(gelu, deg, 16.0)
    ct = ctx.encrypt(ctx.encode(x / 16.0 if pre else x), 5)
    for i in range(3): y = ctx.eval_chebyshev(ct, co, 16.0, pre)
    ctx.synchronize()
    t = time.perf_counter(); n = 10
    for i in range(n): y = ctx.eval_chebyshev(ct, co, 16.0, pre)
    ctx.synchronize(); dt = (time.perf_counter() - t) / n
    print(f"deg {deg} pre {pre}: {dt*1e3:.2f} ms  err {np.abs(ctx.decrypt(y) - po.cheb_eval(co, 16.0, x)).max():.2e}")
a = ctx.encrypt(ctx.encode(x / 16), 5)
for i in range(3): m = ctx.mul(a, a)
ctx.synchronize(); t = time.perf_counter()
for i in range(50): m = ctx.mul(a, a)
ctx.synchronize(); print(f"mul L=12: {(time.perf_counter()-t)/50*1e3:.3f} ms")
pt = ctx.encode(np.full(ctx.slots, 0.3), scale=float(ctx.primes[12]))
ctx.synchronize(); t = time.perf_counter()
for i in range(50): pt = ctx.encode(np.full(ctx.slots, 0.3), scale=float(ctx.primes[12]))
ctx.synchronize(); print(f"encode const: {(time.perf_counter()-t)/50*1e3:.3f} ms")
