#!/bin/bash
# swap-AB transposed TMA store: parity, then bench + debug counters of the skinny shape
O=gpurun_out/r02s3b
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "swap or deepbench or smoke or padding or fallback or ragged or split" > $O/pytest_swap.log 2>&1; echo "rc=$?" >> $O/pytest_swap.log
timeout 300 python bench.py --workload deepbench_b --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_deepbench_b.json 2> $O/bench.err
for shp in "35 8464 2560 rr 0 0 0" "35 8464 2560 rc 0 0 0"; do
  set -- $shp
  echo "== $shp" >> $O/dbg.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg.txt 2>&1
done
