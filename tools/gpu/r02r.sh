set -u
OUT=gpurun_out/r02r; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
CMD4="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
CMD5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
$CMD4 > $OUT/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_smem -s 3 -c 1 -o $OUT/prof_c4 $CMD4 > $OUT/ncu4.log 2>&1; echo ncu4 $?
$CMD5 > $OUT/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fsb_lt_band4 -s 3 -c 1 -o $OUT/prof_c5 $CMD5 > $OUT/ncu5.log 2>&1; echo ncu5 $?
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv --log-file $OUT/launches_c4.csv $CMD4 > $OUT/ncu_l4.log 2>&1; echo l4 $?
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 400 --csv --log-file $OUT/launches_c5.csv $CMD5 > $OUT/ncu_l5.log 2>&1; echo l5 $?
