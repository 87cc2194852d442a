#!/bin/bash
# config-4 e2e (fs_encode_host) check: PCIe link, knobs
set -u
OUT=gpurun_out/s3t; mkdir -p $OUT
python tools/gpu/pcie_bw.py 2>&1 | tail -3
for env in "FSB_PAIR_GLOBAL=1" "FSB_PAIR_GLOBAL=0" "FSB_TMEM_HEADS=0" "FSB_PAIR_GLOBAL=1"; do
  echo "== $env $(env $env python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])")"
done 2>&1 | tee $OUT/e2e.txt
