#!/bin/bash
# Dev experiment: sustained time + DRAM/L2 traffic per kernel configuration.
for sz in ${SIZES:-8192 4096}; do for cfg in "256 2" "512 2"; do for lay in rr cc; do
  set -- $cfg
  r=$(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ge_fused -s 2 -c 1 --csv python scripts/one_call.py $sz $sz $sz $lay $1 $2 3 2>/dev/null | grep -E "__" | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')
  t=$(python scripts/timed.py $sz $sz $sz $lay $1 $2 300)
  echo "n=$sz bn=$1 cg=$2 $lay | $t | $r"
done; done; done
