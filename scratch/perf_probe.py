import sys, time, numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import pyoracle as po
from paper_2306_09189_b200 import Context
cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfgname]
ctx = Context.from_config(cfgname)
ctx.keygen(7)
c,m,k = geo
img, filt = po.make_inputs(c,m,k,c,1000,2000, 2 if cfgname=="cfg4" else 0)
t=time.time(); layer = ctx.conv_layer(c, c, m, k, filt); print("layer", time.time()-t)
t=time.time(); ctx.gen_galois_keys(layer.steps()); print("keys", time.time()-t)
ct = ctx.encrypt(ctx.encode(img), 9000)
ref = po.emu_conv_slots(c,m,k,c,c*m*m,img,filt,2)
for plan in (1,2):
    out = ctx.conv2d(ct, layer, plan); ctx.synchronize()
    print("err", np.abs(ctx.decrypt(out) - ref).max())
    t=time.time()
    for _ in range(iters):
        out = ctx.conv2d(ct, layer, plan)
    ctx.synchronize()
    dt=(time.time()-t)/iters
    print(cfgname, "plan", plan, "ms/conv", dt*1e3, "conv/s", 1/dt)
