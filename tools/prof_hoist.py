"""Per-kernel-class profile of fhe_rotate_hoisted_batch_into (cfg3, B ciphertexts x the 8 stencil shifts)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = Context.from_config("cfg3")
ctx.keygen(7)
st = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(st)
rng = np.random.default_rng(0)
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, 16384)), 9000 + i) for i in range(B)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8)), 1) for _ in range(B * len(st))]
for _ in range(2):
    ctx.rotate_hoisted_batch_into(cts, st, outs)
ctx.synchronize()
n = 4
ctx.timer_start()
for _ in range(n):
    ctx.rotate_hoisted_batch_into(cts, st, outs)
ms = ctx.timer_stop() / n
ctx.prof_reset()
ctx.prof_enable(True)
for _ in range(n):
    ctx.rotate_hoisted_batch_into(cts, st, outs)
ctx.prof_enable(False)
parts = []
for cl in ["ntt", "ntt_modup", "ntt_moddown", "ks_multi", "moddown", "ks_inner"]:
    t, l, by = ctx.prof_get_bytes(cl)
    if l:
        parts.append(f"{cl}={t / n:.3f}ms/{l // n}L ({by / (t * 1e-3) / 1e9:.0f}GB/s)")
nrot = B * len(st)
print(f"B={B}: {ms:.3f} ms per call, {ms / nrot * 1e3:.1f} us/rot ({nrot / ms * 1e3:.0f} rot/s): " + " ".join(parts))
