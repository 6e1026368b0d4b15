#!/bin/bash
# A/B of the single-launch cluster NTT (k_ntt_fused) against the two-launch transform, and of its
# occupancy variants (tools/var/nttf*/): conv and hoisted-rotation timings with output hashes.
mkdir -p gpurun_out
OUT=gpurun_out/ab_nttf.txt
: > $OUT
run() {
  echo "== $1" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 5 cfg1 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-400 >> $OUT
  timeout 300 python tools/prof_hoist.py 1 2>&1 | cut -c1-120 >> $OUT
}
run "two launches (default)"
FHE_NTT_FUSED=1 run "fused, MINB=1"
for v in tools/var/nttf*/; do FHE_NTT_FUSED=1 FHECONV_LIB=$v/libfheconv.so run "fused $(basename $v)"; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_gpu_single_row_shards.py -m gpu -x -q --timeout 300 >> $OUT 2>&1
echo "pytest exit $?" >> $OUT
