#!/bin/bash
# env knobs re-checked on the final kernel (config 4, 256 stripes back to back)
set -u
OUT=gpurun_out/s3x; mkdir -p $OUT
for r in 1 2; do
for env in "X=0" "FSB_WAIT_NS=200" "FSB_WAIT_NS=1000" "FSB_PRECODE_WARPS=4" "FSB_PRECODE_WARPS=5" "FSB_TAIL_SINGLES=0" "FSB_ITEM_OVERHEAD=10" "FSB_ITEM_OVERHEAD=14"; do
  echo "== $env $(env $env python tools/gpu/stripe_sweep.py 200 256)"
done; done 2>&1 | tee $OUT/sweep.txt
