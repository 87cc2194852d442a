set -u
mkdir -p gpurun_out/r02k
B="-DFSB_BAND_BT=64"
VARIANTS="b4=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 $B;b4pol=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 $B -DFSB_BAND_POLICY=1;b3=-DFSB_BAND_V4=3 -DFSB_BAND4_MINB=6 $B;b6=-DFSB_BAND_V4=6 -DFSB_BAND4_MINB=4 $B;b4l2=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 $B -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02k/ab.txt
# ncu of the b4 kernel (config 5)
export FSB_LIB=$PWD/gpurun_out/ab/libb4.so
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fsb_lt_band4 -s 3 -c 1 -o gpurun_out/r02k/prof_c5_b4 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/r02k/ncu.log 2>&1; echo ncu rc=$?
