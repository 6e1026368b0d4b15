#!/bin/bash
# ncu --set full of the big forward NTT passes of one batched cfg3 conv (16 ciphertexts, approach 5):
# the first launch of k_ntt_cols and of k_ntt_rows with the ModUp grid; summaries in gpurun_out/ntt_*_summary.txt
mkdir -p gpurun_out
python tools/one_conv.py 16 5 || exit 1
for k in k_ntt_cols k_ntt_rows; do
  ncu -f --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 3 -o gpurun_out/$k python tools/one_conv.py 16 5 > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${k}_sass.csv 2>&1
  python tools/ncu_summary.py $k > gpurun_out/ntt_${k}_summary.txt 2>&1
  rm -f gpurun_out/${k}_sass.csv gpurun_out/${k}_raw.csv
done
