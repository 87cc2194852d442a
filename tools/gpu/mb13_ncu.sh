nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb13 tools/microbench/mb13.cu
timeout 600 ncu --clock-control none -k regex:gather_dup --launch-skip 0 --launch-count 22 \
  --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,sm__cycles_elapsed.avg,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
  --csv /tmp/mb13 > gpurun_out/mb13_ncu.csv 2>&1
tail -5 gpurun_out/mb13_ncu.csv
