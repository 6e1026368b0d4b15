#!/bin/bash
# A/B of the NTT row phase with shared-memory twiddles reused over R rows (FHE_NTT_TWR = 0 (off), 2, 4, 8, 16).
mkdir -p gpurun_out
OUT=gpurun_out/ab_twr.txt
: > $OUT
for r in 0 2 4 8 16; do
  export FHE_NTT_TWR=$r
  echo "== FHE_NTT_TWR=$r" >> $OUT
  timeout 300 python tools/ab_conv.py 16 5 cfg3 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 5 cfg1 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 8 5 cfg4 >> $OUT 2>&1
  timeout 300 python tools/ab_conv.py 16 2 cfg3 >> $OUT 2>&1
  timeout 300 python tools/prof_hoist.py 16 2>&1 | cut -c1-300 >> $OUT
done
unset FHE_NTT_TWR
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_ntt_cluster.py tests/test_gpu_single_row_shards.py -m gpu -x -q --timeout 300 >> $OUT 2>&1
echo "pytest exit $?" >> $OUT
