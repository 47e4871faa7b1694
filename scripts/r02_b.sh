#!/bin/bash
# Round-2 GPU pass B: new parity tests, new bench (HBM roofline, 256^3, sharded batch at N=1),
# debug-stat counters on the skinny shape, racecheck CG=1 vs CG=2, 256^3 ncu kernel durations.
O=gpurun_out/r02b
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in square256 deepbench_b deepbench_a batched64x2048 prologue4096; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
for cfg in "128 1 0" "64 1 0" "128 1 1" "256 1 0" "64 1 1"; do
  set -- $cfg
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py 35 8457 2560 rr $1 $2 $3 >> $O/dbg_skinny.txt 2>&1
done
for cg in 1 2; do
  echo "== racecheck tile_n=256 cta_group=$cg" >> $O/racecheck_cg.txt
  timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python scripts/one_call.py 300 520 200 rr 256 $cg 1 >> $O/racecheck_cg.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_square256.csv \
  python bench.py --workload square256 --steps 5 --warmup 3 --no-cpu-baseline --no-comparators --e2e-steps 0 > $O/bench_square256_ncu.log 2>&1
ls -la $O
