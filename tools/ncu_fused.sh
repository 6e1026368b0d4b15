#!/bin/bash
# ncu --set full of the batched fused baby-step kernel (cfg3, 16 ciphertexts, approach 5), source-level counters
set -x
mkdir -p gpurun_out
python tools/one_conv.py 16 5 || exit 1
ncu -f --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bsgs_fused -c 1 -o gpurun_out/fused16 python tools/one_conv.py 16 5 > gpurun_out/ncu_f16.log 2>&1
ncu -i gpurun_out/fused16.ncu-rep --page raw --csv > gpurun_out/fused16_raw.csv 2>&1
ncu -i gpurun_out/fused16.ncu-rep --page source --csv --print-source sass > gpurun_out/fused16_sass.csv 2>&1
ncu -i gpurun_out/fused16.ncu-rep --page details --csv > gpurun_out/fused16_details.csv 2>&1
ls -la gpurun_out
