#!/bin/bash
# L2 prefetch of the next tile (cp.async.bulk.prefetch.tensor) in the SMEM kernel: GPU tests, A/B
set -u
OUT=gpurun_out/s3f; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x -k "smem or parity or stripes" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for r in 1 2 3; do
for L in head pf0 pf1; do
  unset FSB_LIB FSB_L2_PREFETCH
  if [ $L = head ]; then export FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_head.so; fi
  if [ $L = pf0 ]; then export FSB_L2_PREFETCH=0; fi
  echo "== $L"; python tools/gpu/stripe_sweep.py 300 16 32 256
done; done 2>&1 | tee $OUT/ab_sweep.txt
unset FSB_LIB FSB_L2_PREFETCH
for c in 6 7; do for pf in 0 1; do echo "== c$c pf$pf"; FSB_L2_PREFETCH=$pf timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done; done 2>&1 | tee -a $OUT/ab_sweep.txt
for pf in 0 1; do echo "== wait share pf$pf"; FSB_L2_PREFETCH=$pf FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=2 python tools/gpu/wait_share.py 2>&1 | tail -3; done 2>&1 | tee -a $OUT/ab_sweep.txt
