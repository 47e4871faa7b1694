#!/bin/bash
O=gpurun_out/r02n
mkdir -p $O
for shp in "1024 1024 1024 rr 64 1" "1024 1024 1024 rr 128 1" "2048 2048 2048 rr 256 1" "2048 2048 2048 rr 128 2" "1024 1024 1024 rr 128 2"; do
  set -- $shp
  echo "== $shp" >> $O/dbg_mma.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ 1 >> $O/dbg_mma.txt 2>&1
done
ls -la $O
