"""One profiled fhe_rotate_hoisted_batch_into call (cfg3, B ciphertexts x the 8 stencil shifts), bracketed by
fhe_profiler_range for ncu --profile-from-start off (tools/ncu_any.sh)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402
from paper_2306_09189_b200.engine import lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = Context.from_config("cfg3")
ctx.keygen(7)
st = [kk * 32 + ll for kk in (-1, 0, 1) for ll in (-1, 0, 1) if kk or ll]
ctx.gen_galois_keys(st)
rng = np.random.default_rng(0)
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, 16384)), 9000 + i) for i in range(B)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8)), 1) for _ in range(B * len(st))]
ctx.rotate_hoisted_batch_into(cts, st, outs)
ctx.synchronize()
lib().fhe_profiler_range(1)
ctx.rotate_hoisted_batch_into(cts, st, outs)
ctx.synchronize()
lib().fhe_profiler_range(0)
