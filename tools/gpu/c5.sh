#!/bin/bash
# Config 5 iteration: build, GPU parity tests, bench configs 5/3/2, one ncu capture of config 5.
TAG=$1
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
for c in 5 3 2; do
  timeout 300 python bench.py --config $c --no-cpu --steps 200 --e2e-steps 0 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
  echo "c$c $(grep -o '"ms_per_step": [0-9.]*' $OUT/bench_c$c.json) $(grep -o '"frac": [0-9.]*' $OUT/bench_c$c.json | head -1)"
done
CMD="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > $OUT/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_lt -s 3 -c 1 -o $OUT/prof_c5 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
