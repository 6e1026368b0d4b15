#!/bin/bash
# ncu --set full of the forward NTT passes used by ModUp (cfg3, 16 ciphertexts, approach 5): all launches
# of one batched conv; the summary picks the longest
mkdir -p gpurun_out
python tools/one_conv.py 16 5 || exit 1
for k in k_ntt_cols k_ntt_rows; do
  ncu -f --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 8 -o gpurun_out/$k python tools/one_conv.py 16 5 > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>&1
done
