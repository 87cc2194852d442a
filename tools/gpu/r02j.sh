set -u
mkdir -p gpurun_out/r02j
VARIANTS="b4=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6;b4bt64=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 -DFSB_BAND_BT=64;b4bt128=-DFSB_BAND_V4=4 -DFSB_BAND4_MINB=6 -DFSB_BAND_BT=128" CONFIGS="5" ROUNDS=3 STEPS=300 CMD='python tools/gpu/check_cfg.py 5 global 2>&1 | tail -1 | tr "\n" " "' bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02j/ab.txt
for r in 4 8 16 32; do echo "rows/warp $r: $(FSB_LIB=$PWD/gpurun_out/ab/libb4.so FSB_BAND_ROWS=$r python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"; done | tee -a gpurun_out/r02j/ab.txt
