#!/bin/bash
# 32-B lanes, warp-split fix: full GPU suite, A/B vs the 16-B-lane build, LPT overhead / split knobs
set -u
OUT=gpurun_out/s3j; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
grep -E "^E .*Error|FAILED" $OUT/pytest_gpu.log | head -5
for r in 1 2; do
for L in head new ov12 ov16 ov24; do
  unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2 FSB_ITEM_OVERHEAD
  case $L in head) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so;; ov12) export FSB_ITEM_OVERHEAD=12;; ov16) export FSB_ITEM_OVERHEAD=16;; ov24) export FSB_ITEM_OVERHEAD=24;; esac
  echo "== $L"; python tools/gpu/stripe_sweep.py 200 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2 FSB_ITEM_OVERHEAD
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=2 python tools/gpu/wait_share.py 2>&1 | tail -2
