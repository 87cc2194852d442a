#!/bin/bash
set -u
mkdir -p gpurun_out/s3b
FSB_EXPERIMENTS=1 python paper_1702_07409_b200/build.py --out $PWD/paper_1702_07409_b200/libfsb_exp.so > /dev/null 2>&1 || echo BUILD FAIL
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=4 python tools/gpu/timeline.py 32 256 2>&1 | tee gpurun_out/s3b/timeline.jsonl
