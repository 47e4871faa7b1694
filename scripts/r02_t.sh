#!/bin/bash
O=gpurun_out/r02t
mkdir -p $O
S=("4096 4096 4096 rr" "4096 4096 4096 rr 256 2" "4096 4096 4096 rr 512 2" "4096 4096 4096 rr 256 1" "4096 4096 4096 cc 256 2" "8192 8192 8192 rr 256 2" "2048 2048 2048 rr 256 2")
for rep in 1 2; do
for v in default xw8; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold --prologue scale_k >> $O/ab.txt 2>&1
done
done
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "8192 8192 8192 rr" "2048 2048 2048 rr" --cold >> $O/noprologue.txt 2>&1
ls -la $O
