#!/bin/bash
# A/B of hoisted rotations and the batched conv: the in-tree build vs every tools/var/<name>/libfheconv.so
for v in "" tools/var/*/; do
  n=${v:-base}; n=$(basename $n)
  if [ -n "$v" ]; then export FHECONV_LIB=$v/libfheconv.so; else unset FHECONV_LIB; fi
  echo -n "$n  "; python tools/ab_conv.py 16 5
  echo -n "$n  "; python tools/prof_hoist.py 16 | cut -c1-60
done
