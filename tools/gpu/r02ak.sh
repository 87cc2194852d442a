# SMEM kernel store addressing (per-tile half offsets, one row x t multiply-add per store): A/B vs the
# previous build (tools/gpu/ab/lib_base.so), parity
set -u
OUT=gpurun_out/r02ak; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for r in 1 2 3; do for lib in base new; do
  if [ $lib = base ]; then export FSB_LIB=$PWD/tools/gpu/ab/lib_base.so; else unset FSB_LIB; fi
  echo "$lib $(for c in 4 6 7 2; do echo -n "c$c $(python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done)"
done; done | tee $OUT/ab.txt
