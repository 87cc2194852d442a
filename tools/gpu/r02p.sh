set -u
OUT=gpurun_out/r02p; mkdir -p $OUT
FSB_EXPERIMENTS=1 python paper_1702_07409_b200/build.py --force --out gpurun_out/ab/libexp.so > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail $OUT/build.log; exit 1; }
for c in 4 6 7; do FSB_LIB=$PWD/gpurun_out/ab/libexp.so FSB_DEBUG=2 python tools/gpu/wait_share.py $c; done | tee $OUT/wait_share.txt
