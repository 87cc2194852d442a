# fsb_lt_win shapes on config 5: window registers (3/4/5 x 32 edges) x rows per window, vs band4
set -u
OUT=gpurun_out/r02z; mkdir -p $OUT gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for v in "5 3 12" "5 4 16" "5 5 20" "5 5 32"; do set -- $v
  FSB_BAND_CFG=$1 FSB_WIN_REGS=$2 FSB_WIN_ROWS=$3 timeout 600 python tools/gpu/check_win.py 5 | sed "s/^/regs$2 rows$3 /"
done | tee $OUT/parity.txt
python paper_1702_07409_b200/build.py --out $PWD/gpurun_out/ab/libl2.so -DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY > $OUT/build_l2.log 2>&1 || tail -3 $OUT/build_l2.log
for round in 1 2 3; do
  for v in "4 3 8" "5 3 12" "5 3 16" "5 4 12" "5 4 16" "5 4 20" "5 5 16" "5 5 20" "5 5 24" "5 5 32"; do set -- $v
    echo "cfg$1 regs$2 rows$3 $(FSB_BAND_CFG=$1 FSB_WIN_REGS=$2 FSB_WIN_ROWS=$3 python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
  for v in "4 3 8" "5 3 16" "5 5 20"; do set -- $v
    echo "L2ONLY cfg$1 regs$2 rows$3 $(FSB_LIB=$PWD/gpurun_out/ab/libl2.so FSB_BAND_CFG=$1 FSB_WIN_REGS=$2 FSB_WIN_ROWS=$3 python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
done | tee $OUT/ab.txt
