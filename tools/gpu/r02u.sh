set -u
OUT=gpurun_out/r02u; mkdir -p $OUT gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
python paper_1702_07409_b200/build.py --force --out gpurun_out/ab/libtssmem.so -DFSB_TS_SMEM_SCHED=1 > $OUT/b2.log 2>&1 || exit 1
FSB_LIB=$PWD/gpurun_out/ab/libtssmem.so FSB_TMEM_SCHED=1 timeout 300 python tools/gpu/check_cfg.py 4 smem | tail -1
for r in 1 2; do
 echo "ts: $(FSB_TMEM_SCHED=1 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
 echo "ts_smem_sched: $(FSB_LIB=$PWD/gpurun_out/ab/libtssmem.so FSB_TMEM_SCHED=1 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
 echo "off: $(FSB_TMEM_SCHED=0 python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"
done | tee $OUT/ab.txt
