set -x
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb13 tools/microbench/mb13.cu && timeout 120 /tmp/mb13 | tee gpurun_out/mb13.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
