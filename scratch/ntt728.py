import sys, ctypes as C
sys.path.insert(0, ".")
from paper_2306_09189_b200 import Context
from paper_2306_09189_b200.engine import lib
ctx = Context.from_config("cfg3")
ms = C.c_float()
assert lib().fhe_bench_ntt(ctx.h, 728, 0, 2, C.byref(ms)) == 0
print(ms.value / 728 * 1e3, "us/row")
