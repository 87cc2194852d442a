# fsb_lt_win with the next-band L2 prefetch (FSB_WIN_PF) on config 5
set -u
OUT=gpurun_out/r02aa; mkdir -p $OUT gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for v in "0 12" "1 12" "1 16"; do set -- $v
  FSB_BAND_CFG=5 FSB_WIN_PF=$1 FSB_WIN_ROWS=$2 timeout 600 python tools/gpu/check_win.py 5 | sed "s/^/pf$1 rows$2 /"
done | tee $OUT/parity.txt
for round in 1 2 3; do
  for v in "4 0 8" "5 0 12" "5 1 12" "5 1 10" "5 1 16" "5 0 10"; do set -- $v
    echo "cfg$1 pf$2 rows$3 $(FSB_BAND_CFG=$1 FSB_WIN_PF=$2 FSB_WIN_ROWS=$3 python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
done | tee $OUT/ab.txt
