# consumer wait between probes of a tile's barriers (FSB_WAIT_NS) on the final build
set -u
OUT=gpurun_out/r02am; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for r in 1 2 3; do for w in 0 100 500 2000; do
  echo "wait$w $(for c in 4 6; do echo -n "c$c $(FSB_WAIT_NS=$w python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done)"
done; done | tee $OUT/ab.txt
