# precode warps per CTA of the SMEM kernel (FSB_PRECODE_WARPS): parity, then same-box A/B
set -u
OUT=gpurun_out/r02aj; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for pw in 4 5 6 7; do for c in 4 6; do FSB_PRECODE_WARPS=$pw timeout 600 python tools/gpu/check_cfg.py $c smem | sed "s/^/pw$pw /"; done; done | tee $OUT/parity.txt
for r in 1 2 3; do for pw in 3 4 5 6; do
  echo "pw$pw $(for c in 4 6 7; do echo -n "c$c $(FSB_PRECODE_WARPS=$pw python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done)"
done; done | tee $OUT/ab.txt
