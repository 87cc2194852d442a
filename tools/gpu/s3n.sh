#!/bin/bash
set -u
OUT=gpurun_out/s3n; mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > $OUT/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_smem -s 3 -c 1 -o $OUT/prof_c4 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=2 python tools/gpu/wait_share.py 2>&1 | tail -1 > $OUT/wait_share.txt
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 python tools/gpu/tile_log.py 256 > $OUT/tile_log_c4.json 2>&1
