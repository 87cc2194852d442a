# window kernel: multi-stripe / ragged-band parity test, random-code stress (encode ranges go through fsb_lt_win)
set -u
OUT=gpurun_out/r02al; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "window" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 1500 python tools/gpu/stress_misc.py 0 300 > $OUT/stress_misc.txt 2>&1; tail -3 $OUT/stress_misc.txt
