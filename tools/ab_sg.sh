#!/bin/bash
# A/B of the sources per CTA of k_bsgs_tma (FHECONV_TMA_SG = 4 / 8 / 16): conv and hoisted timings with hashes.
mkdir -p gpurun_out
OUT=gpurun_out/ab_sg.txt
: > $OUT
for sg in 4 8 16; do
  export FHECONV_TMA_SG=$sg
  echo "== FHECONV_TMA_SG=$sg" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 32 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 5 cfg1 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 8 5 cfg4 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 2 cfg3 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-300 >> $OUT
done
unset FHECONV_TMA_SG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_gpu_parity_r2.py tests/test_gpu_ntt_cluster.py -m gpu -x -q --timeout 300 >> $OUT 2>&1
echo "pytest exit $?" >> $OUT
