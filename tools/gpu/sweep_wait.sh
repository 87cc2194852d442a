#!/bin/bash
# Sweep of the consumer tile-wait backoff (FSB_WAIT_NS) on the config-4 bench.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/sweepw
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for ns in 32 100 200 400 1000; do
  FSB_WAIT_NS=$ns python bench.py --no-cpu --e2e-steps 0 --steps 500 > gpurun_out/sweepw/ns$ns.json 2>&1
  echo "ns=$ns $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweepw/ns$ns.json)"
done
