#!/bin/bash
# cross-class matching of the leftover rows (FSB_PAIR_GLOBAL=1) vs within-class extremes
set -u
OUT=gpurun_out/s3s; mkdir -p $OUT
for r in 1 2 3; do for pg in 0 1; do
  echo "== pg$pg $(FSB_PAIR_GLOBAL=$pg python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/ab_sweep.txt
for c in 6 7; do for pg in 0 1; do
  echo "== c$c pg$pg $(FSB_PAIR_GLOBAL=$pg timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
FSB_PAIR_GLOBAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline or smem or stripes" 2>&1 | tail -2 | tee -a $OUT/ab_sweep.txt
