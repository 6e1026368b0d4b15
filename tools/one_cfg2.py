"""One keyed rotation of NCT cfg2 ciphertexts bracketed by fhe_profiler_range (ncu --profile-from-start off)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context  # noqa: E402
from paper_2306_09189_b200.engine import lib  # noqa: E402

NCT = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = Context.from_config("cfg2")
ctx.keygen(7)
ctx.gen_galois_keys([1, 2])
rng = np.random.default_rng(0)
cts = [ctx.encrypt(ctx.encode(rng.uniform(-1, 1, ctx.slots)), 9000 + i) for i in range(NCT)]
outs = [ctx.encrypt(ctx.encode(np.zeros(8)), 1) for _ in range(NCT)]
ctx.rotate_hoisted_batch_into(cts, [1], outs)
ctx.rotate_hoisted_batch_into(cts, [2], outs)
ctx.synchronize()
lib().fhe_profiler_range(1)
ctx.rotate_hoisted_batch_into(cts, [1], outs)
ctx.synchronize()
lib().fhe_profiler_range(0)
