#!/bin/bash
O=gpurun_out/r02i
mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in square256 square1024 square2048 square4096 deepbench_a deepbench_b prologue4096 hadamard4096 batched64x2048; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
for shp in "35 8464 2560 rr 0 0 0" "1024 1024 1024 rr 0 0 0"; do
  set -- $shp
  echo "== $shp" >> $O/dbg_timeline.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg_timeline.txt 2>&1
done
ls -la $O
