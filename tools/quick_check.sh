#!/bin/bash
# Quick GPU check of the in-tree build: parity subset, then conv and hoisted-rotation timings
# with output hashes (tools/ab_conv.py; hashes must equal the previous build's for bit-identical residues).
mkdir -p gpurun_out
OUT=gpurun_out/quick.txt
: > $OUT
timeout 900 python -m pytest ${PYTEST_FILES:-tests/test_gpu_parity.py tests/test_gpu_tma.py} -m gpu -x -q --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} >> $OUT 2>&1
echo "pytest exit $?" >> $OUT
for a in "16 5 cfg3" "1 5 cfg3" "16 5 cfg1" "4 5 cfg4" "16 2 cfg3"; do timeout 300 python tools/ab_conv.py $a >> $OUT 2>&1; done
timeout 300 python tools/prof_hoist.py 16 >> $OUT 2>&1
timeout 300 python tools/prof_hoist.py 1 >> $OUT 2>&1
