#!/bin/bash
O=gpurun_out/r02j
mkdir -p $O
S=("35 8464 2560 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "5124 704 2048 rr")
timeout 300 python scripts/timed_multi.py "${S[@]}" --cold > $O/alt.txt 2>&1
timeout 300 python scripts/timed_multi.py "${S[@]}" --cold --alt rc >> $O/alt.txt 2>&1
timeout 300 python scripts/timed_multi.py "35 8464 2560 rc" "1024 1024 1024 rc" "2048 2048 2048 rc" "5124 704 2048 rc" --cold >> $O/alt.txt 2>&1
for shp in "4096 4096 4096 rr 0 0 0 0 scale_k" "4096 4096 4096 rr 256 2 0 0 scale_k"; do
  set -- $shp
  echo "== $shp" >> $O/dbg_prologue.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg_prologue.txt 2>&1
done
for g in 1 2 4 8 16 32 64; do
  echo "== group_m $g" >> $O/group.txt
  GE_GROUP_M=$g timeout 300 python scripts/timed_multi.py "8192 8192 8192 rr" "4096 4096 4096 rr" "8192 8192 8192 cc" --cold --iters 100 >> $O/group.txt 2>&1
done
ls -la $O
