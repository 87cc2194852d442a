set -u
mkdir -p gpurun_out/r02h
VARIANTS="base=;b3_bt64=-DFSB_BAND_V3=32 -DFSB_BAND_BT=64;b3_bt128=-DFSB_BAND_V3=16 -DFSB_BAND_BT=128;b3_bt64l2=-DFSB_BAND_V3=32 -DFSB_BAND_BT=64 -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02h/ab.txt
