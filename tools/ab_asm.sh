#!/bin/bash
# A/B of the assembly kernel: default build and ablibs/*.so (GPU box).
out=gpurun_out/ab_asm.txt
: > $out
echo "== default" >> $out
timeout 300 python tools/asmbench.py $1 >> $out 2>&1
for lib in ablibs/*.so; do
  [ -e "$lib" ] || continue
  echo "== $lib" >> $out
  FB_LIB=$PWD/$lib timeout 300 python tools/asmbench.py $1 >> $out 2>&1
done
