#!/bin/bash
# Dev experiment: MMA-loop boundary variants (GE_DEBUG_FLAGS) vs tensor-pipe activity.
for f in 0 1 2 3; do for cfg in "512 2" "256 2"; do set -- $cfg
  r=$(GE_DEBUG_FLAGS=$f ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ge_fused -s 2 -c 1 --csv python scripts/one_call.py 8192 8192 8192 rr $1 $2 3 2>/dev/null | grep -E "__" | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')
  echo "flags=$f bn=$1 cg=$2 $r"
done; done
