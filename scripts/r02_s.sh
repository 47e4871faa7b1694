#!/bin/bash
O=gpurun_out/r02s
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in square256 square1024 square2048 square4096 deepbench_a deepbench_b prologue4096 hadamard4096; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
ls -la $O
