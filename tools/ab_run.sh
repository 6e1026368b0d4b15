#!/bin/bash
# A/B: the in-tree build vs every tools/var/<name>/libfheconv.so, batch sizes given as args
for B in "$@"; do
  echo -n "base  "; python tools/ab_conv.py $B 5
  for v in tools/var/*/; do echo -n "$(basename $v)  "; FHECONV_LIB=$v/libfheconv.so python tools/ab_conv.py $B 5; done
done
