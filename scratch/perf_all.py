import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfg]
ctx = Context.from_config(cfg); ctx.keygen(7)
c,m,k = geo
rng = np.random.default_rng(0)
img = rng.uniform(-1,1,c*m*m); w = rng.uniform(-1,1,c*c*k*k)
layer = ctx.conv_layer(c,c,m,k,w); ctx.gen_galois_keys(layer.steps())
ct = ctx.encrypt(ctx.encode(img), 9000)
out = ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1)
classes = ["conv_mac", "ks_multi", "pt_matvec", "ntt", "ntt_modup", "ntt_moddown", "ks_inner", "moddown", "rescale"]
for ap in (1,2,3,4):
    for _ in range(3): ctx.conv2d_into(ct, layer, ap, out)
    ctx.synchronize()
    n = 10
    ctx.timer_start()
    for _ in range(n): ctx.conv2d_into(ct, layer, ap, out)
    ms = ctx.timer_stop()/n
    ctx.prof_reset(); ctx.prof_enable(True)
    for _ in range(n): ctx.conv2d_into(ct, layer, ap, out)
    ctx.prof_enable(False)
    br = {cl: round(ctx.prof_get(cl)[0]/n, 3) for cl in classes}
    print(cfg, "approach", ap, f"{ms:.3f} ms/conv  {1e3/ms:.1f} conv/s", br)
