set -u
mkdir -p gpurun_out/r02d
VARIANTS="base=;rows1_8_4=-DFSB_BAND_ROWS_KERNEL=1 -DFSB_ROWS_UNROLL=8 -DFSB_ROWS_MINB=4;rows1_6_5=-DFSB_BAND_ROWS_KERNEL=1 -DFSB_ROWS_UNROLL=6 -DFSB_ROWS_MINB=5;rows2_4_4=-DFSB_BAND_ROWS_KERNEL=2 -DFSB_ROWS_UNROLL=4 -DFSB_ROWS_MINB=4;band2_1_4_4=-DFSB_BAND_V2=1 -DFSB_BAND2_B=4 -DFSB_BAND2_MINB=4" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02d/ab_rows.txt
