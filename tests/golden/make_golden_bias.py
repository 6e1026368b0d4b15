"""Generates tests/golden/golden_bias.npz: convolutions WITH bias and output_scale
from the UNMODIFIED reference (conv_plan / convolve, conv.hpp:46-68; bias_plain
conv.cpp:87-94 and the channel-shard bias conv.cpp:344).

Run in the container that has /root/reference (the GPU box does not):
    make -C oracle && python tests/golden/make_golden_bias.py

Inputs come from the reference's own test helpers (tests/helpers.hpp:13-27);
the bias vectors are seeded numpy draws stored beside the outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

# name: (c, m, kappa, c_out, seed_img, seed_filt, weight_kind, s, plan, output_scale, bias_seed)
BIAS_CASES = {
    "bias_cfg1_a2": (4, 32, 3, 4, 1000, 2000, 0, 4096, 2, 0.5, 3000),
    "bias_cfg1_a1": (4, 32, 3, 4, 1000, 2000, 0, 4096, 1, 1.0, 3001),
    "bias_cfg3_a2": (16, 32, 3, 16, 1001, 2001, 0, 16384, 2, 0.25, 3002),
    "bias_ms_cfg1_c4to8": (4, 32, 3, 8, 1012, 2012, 0, 4096, 0, 0.5, 3003),   # image shards, n_out = 2
    "bias_ms_cfg1_c8": (8, 32, 3, 8, 1010, 2010, 0, 4096, 0, 2.0, 3004),       # t = 2, n_out = 2
    "bias_cs_cfg1_c2m128": (2, 128, 3, 2, 1020, 2020, 0, 4096, 0, 0.5, 3005),  # channel shards, pc = 4
}


def main():
    out = {}
    for name, (c, m, k, co, si, sf, wk, s, plan, osc, bs) in BIAS_CASES.items():
        img, filt = po.make_inputs(c, m, k, co, si, sf, wk, use_ref=True)
        bias = np.random.default_rng(bs).uniform(-0.5, 0.5, co)
        slots, ledger = po.ref_conv_biased(c, m, k, co, img, filt, plan, s, bias, osc)
        out[f"{name}/params"] = np.array([c, m, k, co, si, sf, wk, s, plan, bs], dtype=np.int64)
        out[f"{name}/output_scale"] = np.array([osc])
        out[f"{name}/bias"] = bias
        out[f"{name}/slots"] = slots
        out[f"{name}/ledger"] = ledger
    np.savez_compressed(os.path.join(HERE, "golden_bias.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
