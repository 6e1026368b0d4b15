import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
ctx = Context.from_config("cfg3"); ctx.keygen(7)
c, m, k = 16, 32, 3
rng = np.random.default_rng(0)
layer = ctx.conv_layer(c, c, m, k, rng.uniform(-1, 1, c*c*k*k)); ctx.gen_galois_keys(layer.steps(5))
lv = layer.level; N = ctx.N
for B in (8, 16):
    cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, c*m*m)), 9000+i) for i in range(B)]
    inw, outw = 2*(lv+1)*N, 2*lv*N
    bufs = []
    for _ in range(2):
        h_in = torch.empty(B*inw, dtype=torch.int64, pin_memory=True); h_out = torch.empty(B*outw, dtype=torch.int64, pin_memory=True)
        hv = h_in.numpy().view(np.uint64)
        for i, x in enumerate(cts): hv[i*inw:(i+1)*inw] = x.residues().ravel()
        bufs.append((h_in, h_out))
    for ch in (2, 4, 8):
        for j in range(2): ctx.conv2d_batch_host(bufs[j&1][0].data_ptr(), B, layer, 5, bufs[j&1][1].data_ptr(), chunk=ch, asynchronous=True)
        ctx.host_wait()
        t = time.perf_counter(); n = 10
        for j in range(n): ctx.conv2d_batch_host(bufs[j&1][0].data_ptr(), B, layer, 5, bufs[j&1][1].data_ptr(), chunk=ch, asynchronous=True)
        ctx.host_wait()
        dt = (time.perf_counter() - t) / n
        print(f"async B={B} chunk={ch}: {dt*1e3:.2f} ms/step {B/dt:.1f} conv/s e2e", flush=True)
