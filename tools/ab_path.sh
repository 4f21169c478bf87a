out=gpurun_out/ab_path.txt
: > $out
echo "== default" >> $out
timeout 300 python tools/pathbench.py --steps 10 >> $out 2>&1
for lib in ablibs/*.so; do echo "== $lib" >> $out; FB_LIB=$PWD/$lib timeout 300 python tools/pathbench.py --steps 10 >> $out 2>&1; done
