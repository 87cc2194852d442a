#!/bin/bash
# random-graph stress of the final SMEM kernel (16 groups, TMEM heads, cross-class pairing) and of
# the other paths, against the oracle
set -u
OUT=gpurun_out/s3v; mkdir -p $OUT
timeout 1500 python tools/gpu/stress_smem.py 0 400 > $OUT/stress_smem.txt 2>&1; tail -3 $OUT/stress_smem.txt
FSB_TMEM_HEADS=0 timeout 900 python tools/gpu/stress_smem.py 400 550 > $OUT/stress_smem_noheads.txt 2>&1; tail -2 $OUT/stress_smem_noheads.txt
timeout 1200 python tools/gpu/stress_misc.py 0 200 > $OUT/stress_misc.txt 2>&1; tail -3 $OUT/stress_misc.txt
