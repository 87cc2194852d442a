set -u
OUT=gpurun_out/r02o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
timeout 600 python tools/gpu/stress_smem.py 0 40 > $OUT/stress_smem.txt 2>&1; tail -2 $OUT/stress_smem.txt
mkdir -p gpurun_out/ab; cp paper_1702_07409_b200/libfsb200.so gpurun_out/ab/libnew.so
python paper_1702_07409_b200/build.py --out gpurun_out/ab/libns2000.so -DFSB_WAIT_NS_DEFAULT=2000 > /dev/null 2>&1
for r in 1 2 3; do for v in new; do echo "$v: $(FSB_LIB=$PWD/gpurun_out/ab/lib$v.so python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')  $(FSB_LIB=$PWD/gpurun_out/ab/lib$v.so python bench.py --config 6 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"; done; echo "old: $(FSB_LIB=$PWD/tools/gpu/libold.so python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*') $(FSB_LIB=$PWD/tools/gpu/libold.so python bench.py --config 6 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"; for ns in 2000 100; do echo "wait_ns $ns: $(FSB_WAIT_NS=$ns python bench.py --config 4 --no-cpu --e2e-steps 0 --steps 300 | grep -o '"ms_per_step": [0-9.]*')"; done; done | tee $OUT/ab.txt
