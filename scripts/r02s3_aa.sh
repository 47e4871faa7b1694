#!/bin/bash
# prologue: no-op transform with the same handshake (noop, results invalid) vs the real transform
O=gpurun_out/r02s3aa
mkdir -p $O
for rep in 1 2; do
for v in default noop; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "8192 8192 8192 rr" --prologue scale_k --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 512 2" "8192 8192 8192 rr" --cold >> $O/ab.txt 2>&1
done
done
cat $O/ab.txt
