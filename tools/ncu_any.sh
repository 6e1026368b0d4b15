#!/bin/bash
# ncu --set full of the first $3 launches matching regex $2 in `python $4...`, summarised to gpurun_out/$1_summary.txt
# (tools/ncu_summary.py); the .ncu-rep is kept in gpurun_out/ for local inspection (ncu -i).
NAME=$1; RX=$2; CNT=$3; shift 3
mkdir -p gpurun_out
python "$@" > /dev/null || exit 1
ncu -f --profile-from-start off --set full --clock-control none --import-source on -k regex:"$RX" -c $CNT -o gpurun_out/$NAME python "$@" > gpurun_out/ncu_$NAME.log 2>&1
ncu -i gpurun_out/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i gpurun_out/$NAME.ncu-rep --page source --csv --print-source sass > gpurun_out/${NAME}_sass.csv 2>&1
python tools/ncu_summary.py $NAME > gpurun_out/${NAME}_summary.txt 2>&1
rm -f gpurun_out/${NAME}_sass.csv gpurun_out/${NAME}_raw.csv; [ -n "$KEEP_REP" ] || rm -f gpurun_out/$NAME.ncu-rep
