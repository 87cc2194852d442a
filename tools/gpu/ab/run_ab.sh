#!/bin/bash
# A/B on one box: build variant A, bench; build variant B, bench; twice.
CS=paper_1702_07409_b200/csrc
for round in 1 2; do
for v in A B; do
  cp tools/gpu/ab/${v}_fsb_kernels.cu $CS/fsb_kernels.cu; cp tools/gpu/ab/${v}_fsb_graph.cpp $CS/fsb_graph.cpp
  [ -f tools/gpu/ab/${v}_fsb_internal.h ] && cp tools/gpu/ab/${v}_fsb_internal.h $CS/fsb_internal.h
  python -c "from paper_1702_07409_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo build $v failed; exit 1; }
  echo -n "$v: "
  if [ -n "${CMD:-}" ]; then eval "$CMD"; fi
  for c in ${CONFIGS:-4 6 7}; do echo -n "c$c $(python bench.py --config $c --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done; echo
done
done
