#!/bin/bash
# Dev: ncu tensor activity + sustained TF/s for the main configs at one size.
sz=${1:-8192}
for cfg in ${CFGS:-512:2 256:2 256:1}; do set -- ${cfg/:/ }
  r=$(ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ge_fused -s 2 -c 1 --csv python scripts/one_call.py $sz $sz $sz rr $1 $2 3 2>/dev/null | grep -E "__" | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}' | sed 's/sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_/tensor_/g')
  t=$(python scripts/timed.py $sz $sz $sz rr $1 $2 300)
  echo "n=$sz bn=$1 cg=$2 | $t | $r"
done
