#!/bin/bash
# Dev experiment: L2 eviction hints x raster group vs DRAM traffic and sustained time (8192^3).
lay=${1:-rr}
for g in 8 16; do for h in 0,0,0 2,0,1 2,1,1 0,0,1 2,2,1 1,2,1; do
  export GE_GROUP_M=$g GE_L2_HINTS=$h
  r=$(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ge_fused -s 2 -c 1 --csv python scripts/one_call.py 8192 8192 8192 $lay 256 2 3 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')
  t=$(python scripts/timed.py 8192 8192 8192 $lay 256 2 300)
  echo "g=$g hints=$h $r $t"
done; done
