#!/bin/bash
# 32-B lanes with the 256-bit store as a template choice: GPU suite, A/B, LPT overhead, configs 6/7
set -u
OUT=gpurun_out/s3k; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
grep -E "^E .*Error|FAILED" $OUT/pytest_gpu.log | head -5
for r in 1 2; do
for L in head ov6 ov12 ov20; do
  unset FSB_LIB FSB_ITEM_OVERHEAD
  case $L in head) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so;; ov12) export FSB_ITEM_OVERHEAD=12;; ov20) export FSB_ITEM_OVERHEAD=20;; esac
  echo "== $L"; python tools/gpu/stripe_sweep.py 200 16 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_ITEM_OVERHEAD
for c in 6 7; do for L in head ov6 ov12; do
  unset FSB_LIB FSB_ITEM_OVERHEAD
  case $L in head) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so;; ov12) export FSB_ITEM_OVERHEAD=12;; esac
  echo "== c$c $L"; timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
