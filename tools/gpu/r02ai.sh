# config 5: per-step time with launches vs a CUDA-graph replay of the same steps; launch list
set -u
OUT=gpurun_out/r02ai; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for r in 1 2; do
  python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 --graph-replay 100 > $OUT/c5_gr$r.json 2>&1
  python -c "import json; d=json.loads(open('$OUT/c5_gr$r.json').read().strip().splitlines()[-1]); print('c5', d['ms_per_step'], d.get('graph_replay'))"
  FSB_PDL=0 python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 300 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c5 nopdl', d['ms_per_step'])"
done | tee $OUT/ab.txt
