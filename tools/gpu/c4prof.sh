#!/bin/bash
# Config 4 SMEM-kernel A/B profile: one ncu --set full capture each with FSB_PAIRED=1 and =0.
TAG=$1
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
for pv in 1 0; do
  FSB_PAIRED=$pv $CMD > $OUT/plain$pv.log 2>&1 && FSB_PAIRED=$pv ncu --set full --clock-control none --import-source on -k regex:fsb_smem -s 3 -c 1 -o $OUT/prof_c4_p$pv $CMD > $OUT/ncu_full$pv.log 2>&1
  echo "ncu p$pv rc=$?"
done
