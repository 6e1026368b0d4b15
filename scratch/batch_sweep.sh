for B in 1 4 8 16 32; do python scratch/perf_b8.py $B 5; done
python scratch/prof5.py cfg1 5; python scratch/prof5.py cfg4 5; python scratch/prof5.py cfg4 4
