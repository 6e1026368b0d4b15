for L in 4 8; do
for KS in 148 296 592 1184; do
for MV in 148 444 1776; do
echo -n "lanes=$L ks=$KS mv=$MV : "
FHECONV_LANES=$L FHECONV_KS_CTAS=$KS FHECONV_MV_CTAS=$MV python scratch/perf_b8.py 8 2>&1 | tail -1
done; done; done
