timeout 300 python -m pytest tests -x -q -m gpu -k "conv and (5 or auto or fused or host or batched)" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python scratch/perf_b8.py 8 5; python scratch/perf_b8.py 1 5
FHECONV_LIB=varlibs/k0/libfheconv.so python scratch/perf_b8.py 8 5; FHECONV_LIB=varlibs/k0/libfheconv.so python scratch/perf_b8.py 1 5
