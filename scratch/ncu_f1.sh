ncu -f --set full --clock-control none --import-source on -k regex:k_bsgs_fused -s 1 -c 1 -o /tmp/fused1 python scratch/one5.py 1 5 > gpurun_out/ncu_f1.log 2>&1
ncu -i /tmp/fused1.ncu-rep --page raw --csv > gpurun_out/fused1_raw.csv 2>&1
ncu -i /tmp/fused1.ncu-rep --page details --csv > gpurun_out/fused1_details.csv 2>&1
