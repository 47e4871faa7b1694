#!/bin/bash
# Dev experiment: raster group size vs DRAM traffic and sustained time (8192^3 rr).
for g in 1 2 4 8 16 32; do
  export GE_GROUP_M=$g
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:ge_fused -s 2 -c 1 --csv python scripts/one_call.py 8192 8192 8192 ${1:-rr} 256 2 3 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v g=$g '{print "group", g, $(NF-2), $(NF-1), $NF}'
  python scripts/timed.py 8192 8192 8192 ${1:-rr} 256 2 200 | sed "s/^/group $g /"
done
