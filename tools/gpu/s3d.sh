#!/bin/bash
# pre_slots staged by the precode warps: GPU tests, same-box A/B against the previous build
set -u
OUT=gpurun_out/s3d; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for r in 1 2 3; do
for L in head new; do
  if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; else unset FSB_LIB; fi
  echo "== $L"; python tools/gpu/stripe_sweep.py 300 8 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=4 python tools/gpu/timeline.py 32 256 > $OUT/timeline.jsonl 2>&1
python -c "
import json
for l in open('$OUT/timeline.jsonl'):
    d=json.loads(l); d.pop('per_cta',None); print(json.dumps(d))"
