set -u
OUT=gpurun_out/r02ab; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for v in 2 3; do FSB_BAND_CFG=5 FSB_WIN_PF=$v timeout 600 python tools/gpu/check_win.py 5 | sed "s/^/pf$v /"; done | tee $OUT/parity.txt
for round in 1 2 3; do
  for v in 0 1 2 3; do
    echo "pf$v $(FSB_BAND_CFG=5 FSB_WIN_PF=$v python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
  done
done | tee $OUT/ab.txt
