#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_LIB=$PWD/paper_2512_20861_b200/libblr_old.so timeout 300 python scripts/decode_prof.py > gpurun_out/decprof_old.txt 2>&1
timeout 300 python scripts/decode_prof.py > gpurun_out/decprof_new.txt 2>&1
