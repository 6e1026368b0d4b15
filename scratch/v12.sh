timeout 300 python -m pytest tests -x -q -m gpu -k "conv and (5 or auto or fused or ledger or zero or host)" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in 1 2; do echo "variant $v"; FHECONV_FUSED_V=$v python scratch/prof5.py cfg3 5; done
