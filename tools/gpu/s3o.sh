#!/bin/bash
set -u
OUT=gpurun_out/s3o; mkdir -p $OUT
for r in 1 2 3; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps20', d['ms_per_step'], d['step_ms_median'], d['roofline']['frac'], d['clocks'])"; done | tee $OUT/driver_like.txt
