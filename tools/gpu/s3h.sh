#!/bin/bash
# 256-row TMA boxes + precode level offsets in shared memory: GPU tests, A/B, tile log
set -u
OUT=gpurun_out/s3h; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for r in 1 2 3; do
for L in head box1 box4; do
  unset FSB_LIB FSB_BOX_UNITS
  if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; fi
  if [ $L = box1 ]; then export FSB_BOX_UNITS=1; fi
  echo "== $L"; python tools/gpu/stripe_sweep.py 300 16 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_BOX_UNITS
for c in 6 7; do for L in head new; do
  unset FSB_LIB; if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; fi
  echo "== c$c $L"; timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
unset FSB_LIB
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 python tools/gpu/tile_log.py 256 2>&1 | tee $OUT/tile_log_c4.json
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 CFG=6 python tools/gpu/tile_log.py 256 2>&1 | tee $OUT/tile_log_c6.json
