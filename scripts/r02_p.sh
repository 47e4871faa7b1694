#!/bin/bash
O=gpurun_out/r02p
mkdir -p $O
for shp in "1024 1024 1024 rr 64 1 1" "1024 1024 1024 rr 128 1 1" "2048 2048 2048 rr 256 2 1" "35 8464 2560 rr 0 0 0" "4096 4096 4096 rr 512 2 1"; do
  set -- $shp
  echo "== $shp" >> $O/dbg.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg.txt 2>&1
done
ls -la $O
