#!/bin/bash
# TMA box count per k-block by layout: rr (A 1 box, B 2 MN-major boxes), rc (1 + 1), cr (2 + 2), cc (2 + 1)
O=gpurun_out/r02s3s
mkdir -p $O
for rep in 1 2; do
timeout 300 python scripts/timed_multi.py "2048 2048 2048 rr" "2048 2048 2048 rc" "2048 2048 2048 cr" "2048 2048 2048 cc" "1024 1024 1024 rr" "1024 1024 1024 rc" "1024 1024 1024 cr" "1024 1024 1024 cc" "5124 704 2048 rr" "5124 704 2048 rc" --cold >> $O/lay.txt 2>&1
timeout 300 python scripts/timed_multi.py "8192 8192 8192 rr" "8192 8192 8192 rc" "8192 8192 8192 cr" "8192 8192 8192 cc" --cold >> $O/lay.txt 2>&1
done
cat $O/lay.txt
