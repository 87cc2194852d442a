#!/bin/bash
# Same-box comparison of N builds of the in-tree sources that differ only in -D macros.
#   VARIANTS="base=;p1=-DFSB_BAND_POLICY=1" CONFIGS="5" ROUNDS=3 STEPS=300 bash tools/gpu/ab/run_multi.sh
# Builds gpurun_out/ab/lib<name>.so per variant, selects each with FSB_LIB, benches each config
# ROUNDS times in rotation (the box-to-box spread is larger than most single-change effects).
set -u
mkdir -p gpurun_out/ab
IFS=';' read -ra VS <<< "$VARIANTS"
names=()
for v in "${VS[@]}"; do
  name=${v%%=*}; defs=${v#*=}
  python paper_1702_07409_b200/build.py --out gpurun_out/ab/lib$name.so $defs > gpurun_out/ab/build_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/ab/build_$name.log; exit 1; }
  names+=("$name")
done
for round in $(seq 1 ${ROUNDS:-3}); do
  for name in "${names[@]}"; do
    export FSB_LIB=$PWD/gpurun_out/ab/lib$name.so
    echo -n "$name: "
    if [ -n "${CMD:-}" ]; then eval "$CMD"; fi
    for c in ${CONFIGS:-4}; do
      echo -n "c$c $(python bench.py --config $c --no-cpu --e2e-steps 0 --steps ${STEPS:-300} ${BENCH_ARGS:-} | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2) "
    done; echo
  done
done
