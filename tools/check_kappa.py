import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from paper_2306_09189_b200 import Context
import pyoracle as po
ctx = Context.from_config("cfg1"); ctx.keygen(7)
for (c, m, k) in [(4, 32, 7), (4, 32, 5), (16, 16, 7), (1, 64, 9)]:
    img, filt = po.make_inputs(c, m, k, c, 7000 + k, 8000 + k, 0)
    layer = ctx.conv_layer(c, c, m, k, filt)
    ctx.gen_galois_keys(layer.steps(0))
    ct = ctx.encrypt(ctx.encode(img), 9000)
    x = img.reshape(c, m, m); w = filt.reshape(c, c, k, k); h = k // 2
    xp = np.pad(x, ((0, 0), (h, h), (h, h)))
    ref = np.zeros((c, m, m))
    for r in range(k):
        for s in range(k):
            ref += np.einsum("fg,fij->gij", w[:, :, r, s], xp[:, r:r + m, s:s + m])
    for ap in (1, 2, 3, 4, 5, 0):
        try:
            out = ctx.conv2d(ct, layer, ap)
            err = np.abs(ctx.decrypt(out)[: c * m * m] - ref.ravel()).max()
            outs = ctx.conv2d_batch([ct, ct], layer, ap)
            errb = np.abs(ctx.decrypt(outs[1])[: c * m * m] - ref.ravel()).max()
            print(c, m, k, ap, f"{err:.2e}", f"{errb:.2e}")
        except Exception as e:
            print(c, m, k, ap, "ERR", e)
