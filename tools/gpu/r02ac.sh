# round-2 window kernel: full GPU tests, config 5 bench line, config 3 (few-wave) windows A/B,
# launch list and one ncu --set full capture of fsb_lt_win
set -u
OUT=gpurun_out/r02ac; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python bench.py --config 5 --no-cpu --steps 300 --e2e-steps 0 > $OUT/bench_c5.json 2>&1; grep -o '"ms_per_step": [0-9.]*' $OUT/bench_c5.json
for r in 1 2 3; do for c in 5 6; do
  echo "c3 cfg$c $(FSB_BAND_CFG=$c python bench.py --config 3 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
done; done | tee $OUT/ab_c3.txt
CMD="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > $OUT/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv $CMD > $OUT/ncu_launch.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_lt -s 3 -c 1 -o $OUT/prof_c5 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"
