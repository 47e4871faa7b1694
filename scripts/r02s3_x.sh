#!/bin/bash
# skinny shape: bench protocol vs timed_multi in one process set
O=gpurun_out/r02s3x
mkdir -p $O
for st in 20 100; do
timeout 300 python bench.py --workload deepbench_b --steps $st --warmup 3 --no-cpu-baseline --no-comparators > $O/b$st.json 2>/dev/null
python scripts/show_bench.py $O/b$st.json
done
timeout 300 python scripts/timed_multi.py "35 8457 2560 rr" "35 8457 2560 rc" "35 8457 2560 rr" --alt rc --cold
timeout 300 python scripts/timed_multi.py "35 8457 2560 rr" "35 8457 2560 rc" --cold
