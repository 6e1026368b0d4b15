python scratch/one5.py 8 5 && \
ncu -f --set full --clock-control none --import-source on -k regex:k_bsgs_fused -s 1 -c 1 -o /tmp/fused8 python scratch/one5.py 8 5 > gpurun_out/ncu5.log 2>&1
ncu -i /tmp/fused8.ncu-rep --page raw --csv > gpurun_out/fused8_raw.csv 2>&1
ncu -i /tmp/fused8.ncu-rep --page details --csv > gpurun_out/fused8_details.csv 2>&1
ncu -i /tmp/fused8.ncu-rep --page source --csv --print-source sass > gpurun_out/fused8_sass.csv 2>&1
ls -la gpurun_out/
