# windows for every GLOBAL call (default): full GPU tests, bench lines of configs 3, 4, 5, smoke
set -u
OUT=gpurun_out/r02ad; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for c in 3 5 4; do timeout 600 python bench.py --config $c --steps 300 > $OUT/bench_c$c.json 2>$OUT/bench_c$c.err; echo "c$c $(grep -o '"ms_per_step": [0-9.]*' $OUT/bench_c$c.json)"; done
