import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2306_09189_b200 import Context
import pyoracle as po
c, m, k = (int(x) for x in sys.argv[1:4])
nb = int(sys.argv[4])
ctx = Context.from_config("cfg1"); ctx.keygen(7)
img, filt = po.make_inputs(c, m, k, c, 7000 + k, 8000 + k, 0)
layer = ctx.conv_layer(c, c, m, k, filt)
ctx.gen_galois_keys(layer.steps(0))
ct = ctx.encrypt(ctx.encode(img), 9000)
outs = ctx.conv2d_batch([ct] * nb, layer, 0)
ctx.synchronize()
print("ok", nb, np.abs(ctx.decrypt(outs[-1])).max())
