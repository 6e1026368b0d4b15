"""Per-kernel-class profile of one keyed rotation of NCT cfg2 ciphertexts (fhe_rotate_hoisted_batch_into with one step:
the building block of BASELINE cfg2's decomposed rotations)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402

NCT = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = Context.from_config("cfg2")
ctx.keygen(7)
ctx.gen_galois_keys([1, 2, 4])
rng = np.random.default_rng(0)
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, ctx.slots)), 9000 + i) for i in range(NCT)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8)), 1) for _ in range(NCT)]
for _ in range(2):
    ctx.rotate_hoisted_batch_into(cts, [1], outs)
ctx.synchronize()
n = 6
ctx.timer_start()
for i in range(n):
    ctx.rotate_hoisted_batch_into(cts, [1 << (i % 3)], outs)
ms = ctx.timer_stop() / n
ctx.prof_reset()
ctx.prof_enable(True)
for i in range(n):
    ctx.rotate_hoisted_batch_into(cts, [1 << (i % 3)], outs)
ctx.prof_enable(False)
parts = []
tot = 0
for cl in ["ntt", "ntt_modup", "ntt_moddown", "ks_multi", "pt_matvec", "bsgs_fused", "ks_inner", "moddown", "rescale"]:
    t, l, by = ctx.prof_get_bytes(cl)
    if l == 0:
        continue
    tot += t
    parts.append(f"{cl}={t / n:.3f}ms/{l // n}L ({by / (t * 1e-3) / 1e9:.0f}GB/s)")
print(f"cfg2 NCT={NCT}: {ms:.3f} ms per keyed rotation of the batch, {1e3 * ms / NCT:.2f} us/ct ({NCT / ms * 1e3:.0f} keyed/s); "
      f"profiled sum {tot / n:.3f}: " + " ".join(parts))
