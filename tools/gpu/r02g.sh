set -u
mkdir -p gpurun_out/r02g
VARIANTS="base=;b3_8=-DFSB_BAND_V3=8;b3p_8=-DFSB_BAND_V3=8 -DFSB_BAND_PERSIST=1;b3p_8l2=-DFSB_BAND_V3=8 -DFSB_BAND_PERSIST=1 -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02g/ab.txt
