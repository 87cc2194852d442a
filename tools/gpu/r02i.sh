set -u
mkdir -p gpurun_out/r02i
VARIANTS="base=;b4_4_6=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6;b4_4_5=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=5;b4_2_8=-DFSB_BAND_V4=2 -DFSB_BAND4_MINB=8;b4_8_4=-DFSB_BAND_V4=8 -DFSB_BAND4_MINB=4;b4_4_6l2=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02i/ab.txt
