set -u
OUT=gpurun_out/r02q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
for r in 1 2; do for ov in 6 10 12 14 18; do echo "overhead $ov: $(for c in 4 6 7; do FSB_ITEM_OVERHEAD=$ov python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2; done | tr '\n' ' ')"; done; done | tee $OUT/ab.txt
