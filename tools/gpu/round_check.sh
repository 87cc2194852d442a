#!/bin/bash
# One gpurun call: GPU tests, microbenchmarks, bench, ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash tools/gpu/round_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)|Thread' >> $OUT/host.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
if [ -f tools/microbench/mb.cu ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench/mb.cu && timeout 120 /tmp/mb > $OUT/microbench.txt 2>&1
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json
for c in 5 6 7 3 2; do
  timeout 300 python bench.py --config $c --no-cpu --steps 200 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; cat $OUT/bench_c$c.json
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fsb_ -s 3 -c 1 -o $OUT/prof_c4 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
for op in decode repair update; do
  timeout 300 python bench.py --op $op --steps 200 > $OUT/bench_$op.json 2> $OUT/bench_$op.err; cat $OUT/bench_$op.json
done
python tools/gpu/partition_share.py 5 200 > $OUT/partition_share.json 2>&1
python tools/gpu/stripe_share.py 300 > $OUT/stripe_share.json 2>&1; cat $OUT/stripe_share.json
# config 5 (GLOBAL path): launch list + one full capture of the LT kernel
C5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$C5 > $OUT/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv --log-file $OUT/launches_c5.csv $C5 > $OUT/ncu_launches_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fsb_lt -s 3 -c 1 -o $OUT/prof_c5 $C5 > $OUT/ncu_full_c5.log 2>&1
echo "ncu c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; tail -c 400 $OUT/bench_reference.json
