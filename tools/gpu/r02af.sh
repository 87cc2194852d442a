# fsb_dpg_win (source windows for the decode / repair level kernel): parity, then same-box A/B
set -u
OUT=gpurun_out/r02af; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_decode.py tests/test_repair.py -q -m gpu -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
run() { env "$@" timeout 300 python bench.py $ARGS --steps 100 --no-cpu --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(\"$ARGS $*\", d[\"ms_per_step\"], d.get(\"checked\"))"; }
for r in 1 2 3; do
  for ARGS in "--op decode" "--op decode --config 4 --eliminate" "--op repair" "--op update"; do
    for w in 0 1 2; do run FSB_DPG_WIN=$w; done
  done
done | tee $OUT/ab.txt
