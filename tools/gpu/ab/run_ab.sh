#!/bin/bash
# Same-box A/B of two builds of the SAME in-tree sources, differing only in -D macros:
#   DEFS_A="" DEFS_B="-DFSB_SOME_VARIANT" CONFIGS="4 5 6" gpurun -- bash tools/gpu/ab/run_ab.sh
# Each variant is built into gpurun_out/ab/lib{A,B}.so and selected with FSB_LIB; csrc/ is never
# modified, so an interrupted run leaves the product source untouched.
set -u
mkdir -p gpurun_out/ab
python paper_1702_07409_b200/build.py --out gpurun_out/ab/libA.so ${DEFS_A:-} > gpurun_out/ab/buildA.log 2>&1 || { echo build A failed; tail gpurun_out/ab/buildA.log; exit 1; }
python paper_1702_07409_b200/build.py --out gpurun_out/ab/libB.so ${DEFS_B:-} > gpurun_out/ab/buildB.log 2>&1 || { echo build B failed; tail gpurun_out/ab/buildB.log; exit 1; }
for round in 1 2 3; do
for v in A B; do
  export FSB_LIB=$PWD/gpurun_out/ab/lib$v.so
  echo -n "$v: "
  if [ -n "${CMD:-}" ]; then eval "$CMD"; fi
  for c in ${CONFIGS:-4 6 7}; do echo -n "c$c $(python bench.py --config $c --no-cpu --e2e-steps 0 --steps ${STEPS:-300} | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "; done; echo
done
done
