# fsb_lt_win (fixed-size edge windows) vs fsb_lt_band4 on config 5: parity, then same-box A/B
set -u
OUT=gpurun_out/r02y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for c in 4 5; do FSB_BAND_CFG=$c timeout 600 python tools/gpu/check_win.py 5; done | tee $OUT/parity.txt
FSB_BAND_CFG=5 FSB_WIN_ROWS=6 timeout 600 python tools/gpu/check_win.py 5 | tee -a $OUT/parity.txt
python paper_1702_07409_b200/build.py --out gpurun_out/ab/libl2.so -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY > $OUT/build_l2.log 2>&1
for round in 1 2 3; do
  for v in "4 8" "5 8" "5 6" "5 12" "5 16"; do
    set -- $v
    echo "cfg$1 rows$2 $(FSB_BAND_CFG=$1 FSB_WIN_ROWS=$2 python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
  for c in 4 5; do
    echo "L2ONLY cfg$c $(FSB_LIB=$PWD/gpurun_out/ab/libl2.so FSB_BAND_CFG=$c python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
done | tee $OUT/ab.txt
