#!/bin/bash
O=gpurun_out/r02s3d
mkdir -p $O
for w in deepbench_b square256 square1024 square2048 deepbench_a; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench.jsonl 2>> $O/bench.err
done
for f in $O/bench.jsonl; do python scripts/show_bench.py $f; done
