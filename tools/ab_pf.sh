#!/bin/bash
# A/B of the prefetching forward row phase (FHE_NTT_PF = 0 (off), 2, 4, 8) on the in-tree build and tools/var/*.
mkdir -p gpurun_out
OUT=gpurun_out/ab_pf.txt
: > $OUT
run() {
  echo "== $1" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 2 cfg3 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-300 >> $OUT
  timeout 300 python tools/prof_cfg2.py 256 2>&1 | cut -c1-200 >> $OUT
}
for r in 0 2 4 8; do FHE_NTT_PF=$r run "in-tree FHE_NTT_PF=$r"; done
for v in tools/var/*/; do for r in 4 8; do FHE_NTT_PF=$r FHECONV_LIB=$v/libfheconv.so run "var $(basename $v) FHE_NTT_PF=$r"; done; done
