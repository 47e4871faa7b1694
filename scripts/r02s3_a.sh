#!/bin/bash
# Re-entry check on the restored build: GPU tests, default bench line, split-K owner phase counters.
O=gpurun_out/r02s3a
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload deepbench_b --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_deepbench_b.json 2>> $O/bench_default.err
for shp in "35 8464 2560 rr 0 0 0" "35 8464 2560 rc 0 0 0"; do
  set -- $shp
  echo "== $shp" >> $O/dbg.txt
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ >> $O/dbg.txt 2>&1
done
ls -la $O
