#!/bin/bash
# A/B of the TMA ring depth of k_bsgs_tma: SG=8 with 3 stages (3 CTAs/SM; in-tree default) vs SG=4 / 2 stages
# (FHECONV_TMA_SG=4) vs SG=8 / 2 stages (tools/var/nst2).
mkdir -p gpurun_out
OUT=gpurun_out/ab_nst.txt
: > $OUT
run() {
  echo "== $1" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 5 cfg1 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 8 5 cfg4 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 2 cfg3 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-300 >> $OUT
}
run "SG=8 NST=3 (default)"
FHECONV_TMA_SG=4 run "SG=4 NST=2"
for v in tools/var/*/; do FHECONV_LIB=$v/libfheconv.so run "var $(basename $v)"; done
