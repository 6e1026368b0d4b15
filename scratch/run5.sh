python -m pytest tests -x -q -m gpu -k "conv and (5 or auto or fused or ledger or zero)" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python scratch/prof5.py cfg3 5
