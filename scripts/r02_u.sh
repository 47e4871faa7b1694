#!/bin/bash
O=gpurun_out/r02u
mkdir -p $O
for rep in 1 2; do
timeout 300 python scripts/timed_multi.py "35 8464 2560 rr" "35 8464 2560 rc" --cold >> $O/skinny.txt 2>&1
for kw in "swap_ab=1,stream_k=1" "swap_ab=2,stream_k=1"; do
  for t in "64 1" "128 1" "256 1"; do
    timeout 300 python scripts/timed_multi.py "35 8464 2560 rr $t" "35 8464 2560 rc $t" --cold --kw "$kw" >> $O/skinny.txt 2>&1
  done
done
timeout 300 python scripts/timed_multi.py "35 8464 2560 rr 128 1" "35 8464 2560 rc 128 1" --cold --kw "swap_ab=1" >> $O/skinny.txt 2>&1
done
ls -la $O
