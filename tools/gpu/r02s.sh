set -u
OUT=gpurun_out/r02s; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail $OUT/build.log; exit 1; }
timeout 600 python tools/gpu/check_cfg.py 4 smem 2>&1 | tail -1
timeout 600 python tools/gpu/check_cfg.py 4 auto 2>&1 | tail -1
for r in 1 2 3; do for ts in 1 0; do echo "tmem_sched=$ts: $(FSB_TMEM_SCHED=$ts python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"; done; done | tee $OUT/ab.txt
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
timeout 600 python tools/gpu/stress_smem.py 0 60 > $OUT/stress_smem.txt 2>&1; tail -2 $OUT/stress_smem.txt
