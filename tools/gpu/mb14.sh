set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb14 tools/microbench/mb14.cu && timeout 300 /tmp/mb14 | tee gpurun_out/mb14.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
