set -u
mkdir -p gpurun_out/r02l
B="-DFSB_BAND_BT=64"
VARIANTS="b4=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 $B;b4dyn=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 $B -DFSB_BAND_DYN=1;b4dyn256=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 -DFSB_BAND_DYN=1" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02l/ab.txt
