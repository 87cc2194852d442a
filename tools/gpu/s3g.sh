#!/bin/bash
set -u
OUT=gpurun_out/s3g; mkdir -p $OUT
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 python tools/gpu/tile_log.py 256 2>&1 | tee $OUT/tile_log_c4.json
FSB_LIB=$PWD/paper_1702_07409_b200/libfsb_exp.so FSB_DEBUG=8 CFG=6 python tools/gpu/tile_log.py 256 2>&1 | tee $OUT/tile_log_c6.json
