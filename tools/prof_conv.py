import sys, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
AP = int(sys.argv[2]) if len(sys.argv) > 2 else 5
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfg]
ctx = Context.from_config(cfg); ctx.keygen(7)
c, m, k = geo
rng = np.random.default_rng(0)
layer = ctx.conv_layer(c, c, m, k, rng.uniform(-1, 1, c*c*k*k)); ctx.gen_galois_keys(layer.steps(AP))
classes = ["ntt", "ntt_modup", "ntt_moddown", "ks_multi", "pt_matvec", "bsgs_fused", "ks_inner", "moddown", "rescale", "conv_mac"]
for B in (int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,16").split(",")):
    cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c*m*m)), 9000+i) for i in range(B)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1) for _ in range(B)]
    for _ in range(2): ctx.conv2d_batch_into(cts, layer, AP, outs)
    ctx.synchronize(); ctx.timer_start()
    n = 4
    for _ in range(n): ctx.conv2d_batch_into(cts, layer, AP, outs)
    ms = ctx.timer_stop() / n
    ctx.prof_reset(); ctx.prof_enable(True)
    for _ in range(n): ctx.conv2d_batch_into(cts, layer, AP, outs)
    ctx.prof_enable(False)
    tot = 0
    parts = []
    for cl in classes:
        t, l, by = ctx.prof_get_bytes(cl)
        if l == 0: continue
        tot += t
        parts.append(f"{cl}={t/n/B:.3f}ms({by/(t*1e-3)/1e9 if t else 0:.0f}GB/s,{l//n}L)")
    print(f"{cfg} ap={AP} B={B}: {ms/B:.3f} ms/conv ({1e3*B/ms:.0f}/s) profiled-sum {tot/n/B:.3f}: " + " ".join(parts), flush=True)
