#!/bin/bash
# split thresholds with the cross-class pairing (config 4, 256 stripes, back to back, same box)
set -u
OUT=gpurun_out/s3u; mkdir -p $OUT
for r in 1 2 3; do
for sp in "60 120" "56 100" "56 104" "52 100"; do
  set -- $sp
  echo "== s$1/$2 $(FSB_SPLIT1=$1 FSB_SPLIT2=$2 python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/sweep.txt
for sp in "60 120" "56 100"; do set -- $sp
  for c in 6 7; do echo "== c$c s$1/$2 $(FSB_SPLIT1=$1 FSB_SPLIT2=$2 timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")"; done
done 2>&1 | tee -a $OUT/sweep.txt
