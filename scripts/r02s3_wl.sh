#!/bin/bash
# workload lines with 100 timed steps (amortises the timed region's fixed graph-start cost)
O=gpurun_out/wl100
mkdir -p $O
for w in square256 square1024 square2048 square4096 deepbench_a deepbench_b prologue4096 hadamard4096 batched64x2048; do
  timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/err.txt
done
python scripts/show_bench.py $O/bench_workloads.jsonl
