# check-free items before the precode wait (FSB_EARLY_ITEMS): parity of the SMEM configs, A/B
set -u
OUT=gpurun_out/r02ag; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for c in 4 6 7; do FSB_EARLY_ITEMS=0 timeout 600 python tools/gpu/check_cfg.py $c smem; done | tee $OUT/parity0.txt
for r in 1 2 3; do for e in 0 1; do
  echo "early$e $(for c in 4 6 7; do echo -n "c$c $(FSB_EARLY_ITEMS=$e python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done)"
done; done | tee $OUT/ab.txt
