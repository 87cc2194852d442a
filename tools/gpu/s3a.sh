#!/bin/bash
# session-3 baseline: quick check (tests + bench c4) and a stripe sweep for the fixed per-launch cost
set -u
bash tools/gpu/quick.sh s3a 0
python tools/gpu/stripe_sweep.py 300 1 2 4 8 16 32 48 64 128 256 > gpurun_out/s3a/stripe_sweep.json 2>&1; cat gpurun_out/s3a/stripe_sweep.json
FSB_TAIL_SINGLES=0 python tools/gpu/stripe_sweep.py 300 32 64 > gpurun_out/s3a/stripe_sweep_nosingles.json 2>&1; cat gpurun_out/s3a/stripe_sweep_nosingles.json
