"""Build a variant libfheconv.so with extra -D flags into tools/var/<name>/ (the sources in $VAR_SOURCES,
default kernels.cu, are recompiled with the flags)."""
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2306_09189_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join("tools", "var", name); os.makedirs(out, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(out, src.replace(".cu", ".o"))
    if src in os.environ.get("VAR_SOURCES", "kernels.cu").split(","):
        subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    else:
        obj = os.path.join(B.CSRC, src.replace(".cu", ".o"))
    objs.append(obj)
subprocess.run([B._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", os.path.join(out, "libfheconv.so"), *objs], check=True)
print(out)
