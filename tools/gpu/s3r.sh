#!/bin/bash
# head prefetch from TMEM (async tcgen05.ld one item ahead): GPU suite, A/B vs libfsb_th.so
set -u
OUT=gpurun_out/s3r; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
grep -E "^E .*Error|FAILED" $OUT/pytest_gpu.log | head -5
for r in 1 2 3; do
for L in th new; do
  unset FSB_LIB; if [ $L = th ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_th.so; fi
  echo "== $L $(python tools/gpu/stripe_sweep.py 200 32 256)"
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB
for c in 6 7; do for L in th new; do
  unset FSB_LIB; if [ $L = th ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_th.so; fi
  echo "== c$c $L"; timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
