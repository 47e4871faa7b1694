#!/bin/bash
O=gpurun_out/r02s3r
mkdir -p $O
for shp in "35 8464 2560 rr 0 0 0" "2048 2048 2048 rr 0 0 0"; do
  set -- $shp
  echo "== $shp" >> $O/dbg.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg.txt 2>&1
done
cat $O/dbg.txt
