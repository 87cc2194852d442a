set -u
mkdir -p gpurun_out/r02c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02c/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c/pytest_gpu.log; tail -3 gpurun_out/r02c/pytest_gpu.log
VARIANTS="base=;p1=-DFSB_BAND_POLICY=1;p2=-DFSB_BAND_POLICY=2;p3=-DFSB_BAND_POLICY=3;l2only=-DFSB_EXPERIMENTS -DFSB_BAND_L2ONLY" CONFIGS="5 3" ROUNDS=3 STEPS=300 bash tools/gpu/ab/run_multi.sh 2>&1 | tee gpurun_out/r02c/ab_band.txt
