#!/bin/bash
# split thresholds x LPT overhead with the TMEM-heads kernel (config 4, 256 stripes, back to back)
set -u
OUT=gpurun_out/s3p; mkdir -p $OUT
for r in 1 2; do
for sp in "60 120" "56 112" "50 100" "52 120" "48 120" "64 128"; do for ov in 12 16; do
  set -- $sp
  echo "== s$1/$2 ov$ov $(FSB_SPLIT1=$1 FSB_SPLIT2=$2 FSB_ITEM_OVERHEAD=$ov python tools/gpu/stripe_sweep.py 200 256)"
done; done; done 2>&1 | tee $OUT/sweep.txt
