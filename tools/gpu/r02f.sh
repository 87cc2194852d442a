set -u
mkdir -p gpurun_out/r02f
VARIANTS="base=;b3_8=-DFSB_BAND_V3=8;b3_7=-DFSB_BAND_V3=7;b3_8l2=-DFSB_BAND_V3=8 -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY;base_l2=-DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02f/ab.txt
