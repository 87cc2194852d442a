#!/bin/bash
# 32-B lanes (16 groups per warp): GPU parity, A/B against the 16-B-lane build, split thresholds
set -u
OUT=gpurun_out/s3i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "smem or stripes or baseline or paired" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
grep -E "Error|assert" $OUT/pytest_gpu.log | head -5
for r in 1 2; do
for L in head s60 s40 s36 s48; do
  unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2
  case $L in head) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so;; s40) export FSB_SPLIT1=40 FSB_SPLIT2=80;; s36) export FSB_SPLIT1=36 FSB_SPLIT2=72;; s48) export FSB_SPLIT1=48 FSB_SPLIT2=48;; esac
  echo "== $L"; python tools/gpu/stripe_sweep.py 200 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_SPLIT1 FSB_SPLIT2
for c in 6 7; do for L in head new; do
  unset FSB_LIB; if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; fi
  echo "== c$c $L"; timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
unset FSB_LIB
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 python tools/gpu/tile_log.py 256 2>&1 | tee $OUT/tile_log_c4.json | head -14
