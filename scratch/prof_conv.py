import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
from paper_2306_09189_b200.engine import lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
approach = int(sys.argv[2]) if len(sys.argv) > 2 else 2
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfg]
ctx = Context.from_config(cfg); ctx.keygen(7)
c,m,k = geo
rng = np.random.default_rng(0)
img = rng.uniform(-1,1,c*m*m); w = rng.uniform(-1,1,c*c*k*k)
layer = ctx.conv_layer(c,c,m,k,w); ctx.gen_galois_keys(layer.steps())
ct = ctx.encrypt(ctx.encode(img), 9000)
out = ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1)
for _ in range(3): ctx.conv2d_into(ct, layer, approach, out)
ctx.synchronize()
t=time.perf_counter()
for _ in range(5): ctx.conv2d_into(ct, layer, approach, out)
ctx.synchronize(); print("ms/conv wall", (time.perf_counter()-t)/5*1e3)
lib().fhe_profiler_range(1)
ctx.conv2d_into(ct, layer, approach, out)
ctx.synchronize()
lib().fhe_profiler_range(0)
