import sys, os, ctypes as C
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
from paper_2306_09189_b200.engine import lib
ctx = Context.from_config("cfg3")
res = []
for rows in (13, 91, 728):
    for inv in (0, 1):
        ms = C.c_float()
        assert lib().fhe_bench_ntt(ctx.h, rows, inv, 20, C.byref(ms)) == 0
        res.append(f"{rows}{'i' if inv else 'f'}:{ms.value*1e3/rows:.3f}")
print(os.environ.get("FHECONV_LIB", "default"), " ".join(res))
