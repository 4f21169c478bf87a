#!/bin/bash
# A/B kernel timing of the default build and the libraries in ablibs/ (GPU box).
#   bash tools/ab.sh "<kbench args for the default build>" ["<kbench args for ablibs>"]
args="$1"
args2="${2:-$1}"
out=gpurun_out/ab.txt
: > $out
echo "== default" >> $out
timeout 300 python tools/kbench.py $args >> $out 2>&1
for lib in ablibs/*.so; do
  [ -e "$lib" ] || continue
  echo "== $lib" >> $out
  FB_LIB=$PWD/$lib timeout 300 python tools/kbench.py $args2 >> $out 2>&1
done
