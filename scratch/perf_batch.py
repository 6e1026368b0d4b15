import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfg]
ctx = Context.from_config(cfg); ctx.keygen(7)
c,m,k = geo
rng = np.random.default_rng(0)
w = rng.uniform(-1,1,c*c*k*k)
layer = ctx.conv_layer(c,c,m,k,w); ctx.gen_galois_keys(layer.steps())
classes = ["ntt", "ntt_modup", "ntt_moddown", "ks_multi", "pt_matvec", "ks_inner", "moddown", "rescale"]
for B in (1, 2, 4, 8, 16):
    cts = [ctx.encrypt(ctx.encode(rng.uniform(-1,1,c*m*m)), 9000+i) for i in range(B)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1) for _ in range(B)]
    for _ in range(2): ctx.conv2d_batch_into(cts, layer, 0, outs)
    ctx.synchronize()
    n = max(2, 16 // B)
    ctx.timer_start()
    for _ in range(n): ctx.conv2d_batch_into(cts, layer, 0, outs)
    ms = ctx.timer_stop() / n
    ctx.prof_reset(); ctx.prof_enable(True)
    for _ in range(n): ctx.conv2d_batch_into(cts, layer, 0, outs)
    ctx.prof_enable(False)
    br = {cl: round(ctx.prof_get(cl)[0] / n / B, 3) for cl in classes}
    print(f"{cfg} batch {B:2d}: {ms:.3f} ms/batch  {ms/B:.3f} ms/conv  {1e3*B/ms:.1f} conv/s  per-conv {br}", flush=True)
