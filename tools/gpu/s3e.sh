#!/bin/bash
# static rounds + dynamic tail: GPU tests, same-box A/B against the previous build, timeline
set -u
OUT=gpurun_out/s3e; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for r in 1 2 3; do
for L in head new; do
  if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; else unset FSB_LIB; fi
  echo "== $L"; python tools/gpu/stripe_sweep.py 300 8 16 32 64 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB
for dd in 1 3; do echo "== new depth $dd"; FSB_DYN_DEPTH=$dd python tools/gpu/stripe_sweep.py 300 8 16 32 64 256; done 2>&1 | tee -a $OUT/ab_sweep.txt
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=4 python tools/gpu/timeline.py 32 256 > $OUT/timeline.jsonl 2>&1
python -c "
import json
for l in open('$OUT/timeline.jsonl'):
    d=json.loads(l); d.pop('per_cta',None); print(json.dumps({k:d[k] for k in ('S','event_us','first_tile_ready','consumer_end_mean','consumer_end_max')}))"
