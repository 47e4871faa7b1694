#!/bin/bash
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "prologue or hadamard or golden" > $O/pytest_prologue.log 2>&1; echo "rc=$?" >> $O/pytest_prologue.log
for w in prologue4096 square4096; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-comparators >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
for shp in "35 8457 2560 rr 0 0 0" "2048 2048 2048 rr 0 0 0" "1024 1024 1024 rr 0 0 0" "256 256 256 rr 0 0 0" "4096 4096 4096 rr 512 2 1"; do
  set -- $shp
  echo "== $shp" >> $O/dbg_timeline.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg_timeline.txt 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:ge_fused -o $O/prologue4096 \
  python scripts/one_call.py 4096 4096 4096 rr 0 0 2 scale_k > $O/prologue4096.log 2>&1
ls -la $O
