# fsb_lt_win32 (1-KB bands, 256-bit gathers) vs fsb_lt_win on config 5 / 3
set -u
OUT=gpurun_out/r02ah; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for v in "1 6" "1 12" "2 6" "2 12"; do set -- $v
  FSB_WIN_V8=$1 FSB_WIN_ROWS=$2 timeout 600 python tools/gpu/check_win.py 5 | sed "s/^/v8=$1 rows$2 /"
  FSB_WIN_V8=$1 FSB_WIN_ROWS=$2 timeout 600 python tools/gpu/check_win.py 3 | sed "s/^/v8=$1 rows$2 /"
done | tee $OUT/parity.txt
for r in 1 2 3; do
  for v in "0 12" "1 6" "1 8" "1 12" "2 6" "2 12"; do set -- $v
    echo "v8=$1 rows$2 $(for c in 5 3; do echo -n "c$c $(FSB_WIN_V8=$1 FSB_WIN_ROWS=$2 python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done)"
  done
done | tee $OUT/ab.txt
