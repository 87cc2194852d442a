#!/bin/bash
# precode warps 1 / 2 / 3 on config 4 (consumers 26 / 25 / 24)
set -u
OUT=gpurun_out/s3y; mkdir -p $OUT
for pw in 1 2 3; do FSB_PRECODE_WARPS=$pw timeout 600 python tools/gpu/check_cfg.py 4 smem 2>&1 | tail -1; done
for r in 1 2; do for pw in 3 2 1; do
  echo "== pw$pw $(FSB_PRECODE_WARPS=$pw python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/sweep.txt
