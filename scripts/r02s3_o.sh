#!/bin/bash
O=gpurun_out/r02s3o
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_dbg.so timeout 300 python scripts/timeline.py "256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "35 8464 2560 rr" > $O/timeline.txt 2>&1
grep -A3 "==\|med" $O/timeline.txt
