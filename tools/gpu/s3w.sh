#!/bin/bash
# 28 consumer warps at 64 registers (1024 threads) vs 24 at 72 (libfsb_final.so)
set -u
OUT=gpurun_out/s3w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline or smem or stripes or paired" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for r in 1 2 3; do
for L in final w28; do
  unset FSB_LIB; if [ $L = final ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_final.so; fi
  echo "== $L $(python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB
for c in 6 7; do for L in final w28; do
  unset FSB_LIB; if [ $L = final ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_final.so; fi
  echo "== c$c $L $(timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
