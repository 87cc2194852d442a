# The bench's N > 1 code path on a one-GPU box: torchrun with 2 and 4 ranks sharing cuda:0 over
# gloo (FSB_BENCH_BACKEND=gloo).  Timings are meaningless (ranks contend for one GPU); the run
# checks that every leg of the N > 1 line (broadcast, shards, max over ranks, gathers, e2e) runs.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mr_build.log 2>&1
for N in 2 4 8; do
  FSB_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 10 --warmup 3 \
    --e2e-steps 2 > gpurun_out/mr_n$N.log 2>&1; echo "N=$N rc=$?"
  FSB_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29610 + N)) bench.py --gpus $N --steps 10 --warmup 3 \
    --config 5 > gpurun_out/mr_c5_n$N.log 2>&1; echo "c5 N=$N rc=$?"
  FSB_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29620 + N)) bench.py --gpus $N --steps 10 --warmup 3 \
    --config 5 --partition cols > gpurun_out/mr_c5c_n$N.log 2>&1; echo "c5 cols N=$N rc=$?"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29630 + N)) bench.py --impl reference --gpus $N --steps 2 --warmup 1 \
    --ref-seconds 4 > gpurun_out/mr_ref_n$N.log 2>&1; echo "ref N=$N rc=$?"
done

tail -c 600 gpurun_out/mr_n2.log
