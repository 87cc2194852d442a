#!/bin/bash
# 16-group kernel: split thresholds with LPT overhead 12, ncu capture, tile log
set -u
OUT=gpurun_out/s3l; mkdir -p $OUT
for r in 1 2; do
for L in head d s56 s64 s48 s40; do
  unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2
  case $L in head) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so;; s56) export FSB_SPLIT1=56 FSB_SPLIT2=112;; s64) export FSB_SPLIT1=64 FSB_SPLIT2=128;; s48) export FSB_SPLIT1=48 FSB_SPLIT2=96;; s40) export FSB_SPLIT1=40 FSB_SPLIT2=80;; esac
  echo "== $L"; python tools/gpu/stripe_sweep.py 200 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 python tools/gpu/tile_log.py 256 2>&1 > $OUT/tile_log_c4.json
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=2 python tools/gpu/wait_share.py 2>&1 | tail -1 > $OUT/wait_share.txt
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > $OUT/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_smem -s 3 -c 1 -o $OUT/prof_c4 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
