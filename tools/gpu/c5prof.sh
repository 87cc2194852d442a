#!/bin/bash
# Config 5 band-kernel profile: bench line, then one ncu --set full capture of fsb_lt_band.
TAG=$1
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
CMD="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
timeout 300 python bench.py --config 5 --no-cpu --steps 200 --e2e-steps 0 > $OUT/bench_c5.json 2>&1
grep -o '"ms_per_step": [0-9.]*' $OUT/bench_c5.json
$CMD > $OUT/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_lt -s 3 -c 1 -o $OUT/prof_c5 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
