set -u
mkdir -p gpurun_out/r02n
VARIANTS="base=;wb=-DFSB_SMEM_ST_WB=1" CONFIGS="4 6 7" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 4 smem 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02n/ab.txt
