for v in varlibs/*; do echo -n "$v: "; FHECONV_LIB=$v/libfheconv.so python scratch/perf_b8.py 8 5 2>&1 | tail -1; done
