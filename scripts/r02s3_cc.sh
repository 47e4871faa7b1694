#!/bin/bash
# MMA warp spinning (no try_wait suspend) on the prologue kernels
O=gpurun_out/r02s3cc
mkdir -p $O
for rep in 1 2 3; do
for v in default spin; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "8192 8192 8192 rr" --prologue scale_k --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" --prologue hadamard --cold >> $O/ab.txt 2>&1
done
done
python scripts/ab_table.py $O/ab.txt
