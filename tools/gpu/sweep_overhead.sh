python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/sweep
for ov in 0 2 4 6 10; do
  FSB_ITEM_OVERHEAD=$ov python bench.py --no-cpu --e2e-steps 0 --steps 500 > gpurun_out/sweep/ov$ov.json 2>&1
  echo "ov=$ov $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep/ov$ov.json)"
done
