#!/bin/bash
# Fast iteration call: build, GPU parity tests, bench config 4 (+ optional extra configs), one ncu capture.
# Usage: bash tools/gpu/quick.sh TAG [ncu:0|1] [configs...]
set -u
TAG=$1; NCU=${2:-1}; shift 2 || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
[ $rc -ne 0 ] && { grep -E "Error|assert|FAIL" $OUT/pytest_gpu.log | head -20; exit 1; }
timeout 600 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err
for c in "$@"; do
  timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; cat $OUT/bench_c$c.json
done
if [ "$NCU" = "1" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
  $CMD > $OUT/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fsb_ -s 3 -c 1 -o $OUT/prof_c4 $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
