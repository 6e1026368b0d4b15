python scratch/ntt728.py || exit 1
for k in rows cols; do
ncu -f --set full --clock-control none --import-source on -k regex:k_ntt_$k -s 2 -c 1 -o /tmp/n$k python scratch/ntt728.py > gpurun_out/ncu_n$k.log 2>&1
ncu -i /tmp/n$k.ncu-rep --page raw --csv > gpurun_out/n${k}_raw.csv 2>&1
ncu -i /tmp/n$k.ncu-rep --page source --csv --print-source sass > gpurun_out/n${k}_sass.csv 2>&1
done
