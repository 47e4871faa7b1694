#!/bin/bash
O=gpurun_out/r02g
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in prologue4096 hadamard4096 square4096 deepbench_b; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
ls -la $O
