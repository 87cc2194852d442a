#!/bin/bash
# check-free items first (FSB_FREE_FIRST=1) vs the final build (libfsb_final.so) and this build with it off
set -u
OUT=gpurun_out/s3z; mkdir -p $OUT
FSB_FREE_FIRST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline or smem or stripes or paired or edge" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for r in 1 2; do
for L in final ff0 ff1; do
  unset FSB_LIB FSB_FREE_FIRST
  case $L in final) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_final.so;; ff1) export FSB_FREE_FIRST=1;; esac
  echo "== $L $(python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/ab_sweep.txt
for c in 6 7; do for L in final ff1; do
  unset FSB_LIB FSB_FREE_FIRST
  case $L in final) export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_final.so;; ff1) export FSB_FREE_FIRST=1;; esac
  echo "== c$c $L $(timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
