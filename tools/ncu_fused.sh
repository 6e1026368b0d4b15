#!/bin/bash
# ncu --set full of the batched fused baby-step kernel (cfg3, 16 ciphertexts, approach 5), source-level counters.
# FHECONV_LIMB=0|1 selects k_bsgs_fused / k_bsgs_limb; $1 = report name (default fused16). Writes a compact
# summary (tools/ncu_summary.py) to gpurun_out/<name>_summary.txt and drops the large CSVs.
set -x
NAME=${1:-fused16}
mkdir -p gpurun_out
python tools/one_conv.py 16 5 || exit 1
ncu -f --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bsgs -c 1 -o gpurun_out/$NAME python tools/one_conv.py 16 5 > gpurun_out/ncu_$NAME.log 2>&1
ncu -i gpurun_out/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i gpurun_out/$NAME.ncu-rep --page source --csv --print-source sass > gpurun_out/${NAME}_sass.csv 2>&1
python tools/ncu_summary.py $NAME > gpurun_out/${NAME}_summary.txt 2>&1
ls -la gpurun_out/${NAME}*; rm -f gpurun_out/${NAME}_sass.csv gpurun_out/${NAME}_raw.csv gpurun_out/${NAME}.ncu-rep
