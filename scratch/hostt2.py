import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
cfg = sys.argv[1]; AP = 5
geo = {"cfg1": (4,32,3), "cfg3": (16,32,3), "cfg4": (8,64,5)}[cfg]
ctx = Context.from_config(cfg); ctx.keygen(7)
c, m, k = geo
rng = np.random.default_rng(0)
layer = ctx.conv_layer(c, c, m, k, rng.uniform(-1, 1, c*c*k*k)); ctx.gen_galois_keys(layer.steps(AP))
for B in (1, 8):
    cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c*m*m)), 9000+i) for i in range(B)]
    outs = [ctx.encrypt(ctx.encode(np.zeros(8), level=ctx.max_level-1), 1) for _ in range(B)]
    for rep in range(8):
        ctx.synchronize()
        t0 = time.perf_counter(); ctx.timer_start()
        ctx.conv2d_batch_into(cts, layer, AP, outs)
        t1 = time.perf_counter()
        ms = ctx.timer_stop(); t2 = time.perf_counter()
        print(f"{cfg} B={B} rep {rep}: enqueue {1e3*(t1-t0):.2f} ms, device {ms:.2f} ms", flush=True)
    ctx.prof_reset(); ctx.prof_enable(True)
    for _ in range(2): ctx.conv2d_batch_into(cts, layer, AP, outs)
    ctx.prof_enable(False)
for trial in range(3):
    ctx.synchronize()
    t0 = time.perf_counter(); ctx.timer_start()
    te = []
    for _ in range(4):
        ctx.conv2d_batch_into(cts, layer, AP, outs); te.append(time.perf_counter())
    ms = ctx.timer_stop()
    print("b2b x4: enqueue", [round(1e3*(te[i]-(te[i-1] if i else t0)),2) for i in range(4)], "device", round(ms, 2), flush=True)
