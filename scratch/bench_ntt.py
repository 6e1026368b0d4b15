import sys, ctypes as C
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
from paper_2306_09189_b200.engine import lib
for cfg in sys.argv[1:] or ["cfg3"]:
    ctx = Context.from_config(cfg)
    for rows in (13, 91, 364, 728):
        for inv in (0, 1):
            ms = C.c_float()
            assert lib().fhe_bench_ntt(ctx.h, rows, inv, 20, C.byref(ms)) == 0
            us = ms.value * 1e3
            gbs = rows * ctx.N * 8 * 4 / (us * 1e-6) / 1e9
            print(f"{cfg} N=2^{ctx.log_n} rows {rows:4d} {'inv' if inv else 'fwd'}: {us:8.1f} us  {us/rows:6.3f} us/row  ({gbs:6.0f} GB/s eff. 2-pass r+w)")
