#!/bin/bash
O=gpurun_out/r02s3w
mkdir -p $O
for shp in "4096 4096 4096 rr 256 2 0 0 relu" "4096 4096 4096 rr 256 2 0 0 scale_k" "4096 4096 4096 cc 256 2 0 0 scale_k"; do
  set -- $shp
  echo "== $shp" >> $O/dbg.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg.txt 2>&1
done
grep -v "^\s*[0-9]*:" $O/dbg.txt | grep "==\|total\|mma_wait\|transform\|MMA warp\|epi_wait\|epi_to\|epi_tile"
