#!/bin/bash
# Sweep of fsb_lt_band's (batch, blocks/SM) variants on configs 5 and 3.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/sweepb
for v in 0 1 2 3 4; do
  for c in 5 3; do
    FSB_BAND_CFG=$v python bench.py --config $c --no-cpu --e2e-steps 0 --steps 200 > gpurun_out/sweepb/v${v}_c$c.json 2>&1
    echo "v=$v c$c $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweepb/v${v}_c$c.json)"
  done
done
