#!/bin/bash
# Round-2 first GPU pass: GPU tests on the round-1 build, bench lines, ncu full captures of the
# kernels VERDICT.md names (skinny 35x8457x2560, SCALE_K prologue 4096^3, 4096^3, batched 64x2048^3).
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in deepbench_b prologue4096 square4096 square2048; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
cap() {  # name M N K lay pro batch
  timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:ge_fused -o $O/$1 \
    python scripts/one_call.py $2 $3 $4 $5 0 0 2 $6 $7 > $O/$1.log 2>&1
}
cap skinny_rr 35 8457 2560 rr none 1
cap skinny_rc 35 8457 2560 rc none 1
cap prologue4096 4096 4096 4096 rr scale_k 1
cap square4096 4096 4096 4096 rr none 1
cap batched64 2048 2048 2048 rr none 64
ls -la $O
