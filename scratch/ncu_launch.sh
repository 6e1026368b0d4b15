python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg2 > gpurun_out/b_short.log 2>&1 || exit 2
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg2 > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
