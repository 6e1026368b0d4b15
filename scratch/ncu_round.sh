set -x
python scratch/one5.py 1 5 || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:k_bsgs_fused -s 2 -c 1 -o /tmp/fused1 python scratch/one5.py 1 5 > gpurun_out/ncu_f1.log 2>&1
ncu -i /tmp/fused1.ncu-rep --page raw --csv > gpurun_out/fused1_raw.csv 2>&1
ncu -i /tmp/fused1.ncu-rep --page details --csv > gpurun_out/fused1_details.csv 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg2 > gpurun_out/b_short.log 2>&1 || exit 2
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg2 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out | head
