#!/bin/bash
# A/B of the in-tree build against every tools/var/<name>/libfheconv.so: conv and hoisted timings with output
# hashes, then the TMA/parity GPU tests on the in-tree build.
mkdir -p gpurun_out
OUT=gpurun_out/ab_var.txt
: > $OUT
run() {
  echo "== $1" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 1 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 5 cfg1 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 8 5 cfg4 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 2 cfg3 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-300 >> $OUT
}
run "in-tree"
for v in tools/var/*/; do FHECONV_LIB=$v/libfheconv.so run "var $(basename $v)"; done
[ -n "$SKIP_TESTS" ] || { timeout 1500 python -m pytest tests/test_gpu_tma.py tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -m gpu -x -q --timeout 300 >> $OUT 2>&1; echo "pytest exit $?" >> $OUT; }
