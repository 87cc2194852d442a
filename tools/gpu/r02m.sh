set -u
OUT=gpurun_out/r02m; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for c in 5 3 4; do timeout 300 python bench.py --config $c --no-cpu --steps 300 --e2e-steps 0 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; python -c "import json; d=json.load(open('$OUT/bench_c$c.json')); print('c$c', d['ms_per_step'], d['roofline']['frac'], d['roofline']['gather']['frac'])"; done
