set -u
OUT=gpurun_out/r02t; mkdir -p $OUT gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
python paper_1702_07409_b200/build.py --force --out gpurun_out/ab/libtma3d.so -DFSB_EXPERIMENTS -DFSB_TS_TMA3D > $OUT/b2.log 2>&1 || exit 1
for r in 1 2; do
 echo "ts5d: $(FSB_TMEM_SCHED=1 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
 echo "ts3d(wrong bytes): $(FSB_LIB=$PWD/gpurun_out/ab/libtma3d.so FSB_TMEM_SCHED=1 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
 echo "off: $(FSB_TMEM_SCHED=0 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
done | tee $OUT/ab.txt
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0"
FSB_TMEM_SCHED=1 $CMD > /dev/null 2>&1 && FSB_TMEM_SCHED=1 ncu --set full --clock-control none --import-source on -k regex:fsb_smem -s 3 -c 1 -o $OUT/prof_ts $CMD > $OUT/ncu.log 2>&1; echo ncu $?
