#!/bin/bash
# A/B of the fused baby-step kernels: k_bsgs_fused (FHECONV_LIMB=0), k_bsgs_limb (FHECONV_TMA=0), k_bsgs_tma
# (default); the output hashes must agree. Args: configs (default cfg3 cfg1 cfg4)
for cfg in ${@:-cfg3 cfg1 cfg4}; do
  for B in 16 1; do
    echo -n "fused "; FHECONV_LIMB=0 python tools/ab_conv.py $B 5 $cfg
    echo -n "limb  "; FHECONV_TMA=0 python tools/ab_conv.py $B 5 $cfg
    echo -n "tma   "; python tools/ab_conv.py $B 5 $cfg
  done
done
