#!/bin/bash
# dynamic tile hand-out: GPU tests, then same-box A/B against the previous build (libfsb_head.so)
set -u
OUT=gpurun_out/s3c; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for r in 1 2; do
for L in head new; do
  if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; else unset FSB_LIB; fi
  echo "== $L"; python tools/gpu/stripe_sweep.py 300 16 32 64 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB
timeout 300 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json | head -c 600; echo
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=4 python tools/gpu/timeline.py 32 256 > $OUT/timeline.jsonl 2>&1
python -c "
import json
for l in open('$OUT/timeline.jsonl'):
    d=json.loads(l); d.pop('per_cta',None); print(json.dumps(d))"
