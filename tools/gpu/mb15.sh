set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb15 tools/microbench/mb15.cu && timeout 300 /tmp/mb15 | tee gpurun_out/mb15.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
