import sys, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
AP = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = Context.from_config("cfg3"); ctx.keygen(7)
c, m, k = 16, 32, 3
rng = np.random.default_rng(0)
layer = ctx.conv_layer(c, c, m, k, rng.uniform(-1, 1, c*c*k*k)); ctx.gen_galois_keys(layer.steps(AP))
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c*m*m)), 9000+i) for i in range(B)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1) for _ in range(B)]
from paper_2306_09189_b200.engine import lib
ctx.conv2d_batch_into(cts, layer, AP, outs)
ctx.synchronize()
lib().fhe_profiler_range(1)  # ncu --profile-from-start off captures only this conv batch
ctx.conv2d_batch_into(cts, layer, AP, outs)
ctx.synchronize()
lib().fhe_profiler_range(0)
