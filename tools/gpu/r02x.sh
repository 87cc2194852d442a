set -u
OUT=gpurun_out/r02x; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tail or config_parity or paired" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for r in 1 2; do for ts in 1 0; do FSB_TAIL_SINGLES=$ts python tools/gpu/stripe_sweep.py 300 5 10 20 32 37 64 128 256; done; done | tee $OUT/sweep.txt
