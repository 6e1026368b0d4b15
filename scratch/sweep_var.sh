for v in varlibs/v2m4 varlibs/v2m3; do echo -n "$v: "; FHECONV_LIB=$v/libfheconv.so python scratch/perf_b8.py 8 5 2>&1 | tail -1; done
